"""Whole-step parity at the BASELINE sizes.

    python scripts/full_parity.py gpu c3 [--out DIR]        # the product path on cuda:0
    python scripts/full_parity.py oracle c3 [--ranks 16]    # the oracle on all host cores
    python scripts/full_parity.py both c3                   # both, then compare

The GPU leg runs one full outer step of the config through the public API
(bench.Problem: inputs generated in HBM by pc_gen_* or uploaded from the host
recipe, then ptl.split_advance) and saves the initial and final state and
the per-cycle report.  The oracle leg runs the slab-decomposed oracle
(oracle/distributed.py: the CPU restatement, one gloo rank per host core,
each rank generating its own slab of the seeded inputs from the host recipes
in configs.py) over the same step and compares, rank by rank:

* inputs: the GPU's initial state == the host recipe, bitwise;
* Delta t_E, and per operator the per-cycle (dt, stages / PCG iterations);
* fields: bitwise for RKL2; relative L2 <= 1e-10 for BE (the PCG inner
  products take their partial sums in another order).

Cases: c2, c3, c4 at their BASELINE sizes; c5r = the C5 recipe (coupled
conduction + viscosity, rho field, 5e4 dt_E -- the bench's own ratio) on a
reduced 128 x 128 x 256 grid; c5vr / c4r = the C5v / C4 recipes as one
whole step on that grid; c3g = C3 advanced with RKG2.  Results: DIR/full_parity_<case>.json.
This is test infrastructure (it executes oracle/), not part of the product.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import sys
import time
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

CASES = {
    "c2": ("c2", None),
    "c3": ("c3", None),
    "c4": ("c4", None),
    "c5r": ("c5", (128, 128, 256)),
    # the C5v recipe (C5's viscosity alone at 5e4 dt_E(viscosity), radial rho) on the C5r grid
    "c5vr": ("c5v", (128, 128, 256)),
    # the C4 recipe (BE + Jacobi PCG under PTL at 1e4 dt_E) as one WHOLE step on the C5r grid: every PTL cycle
    # and PCG solve of the step (the BASELINE-size C4 step is 576 iterations, hours of oracle time)
    "c4r": ("c4", (128, 128, 256)),
    # C3 at BASELINE size advanced with RKG2 instead of RKL2 (the second STS family, whole step)
    "c3g": ("c3", None),
    # tiny versions for the CPU self-check of this script (leg "fake")
    "c2t": ("c2", (12, 8, 16)),
    "c3t": ("c3", (14, 10, 32)),
    "c3gt": ("c3", (14, 10, 32)),
    "c4t": ("c4", (14, 10, 32)),
    "c5t": ("c5", (14, 10, 32)),
    "c5vt": ("c5v", (14, 10, 32)),
}
SCHEME = {"c3g": "rkg2", "c3gt": "rkg2"}  # scheme overrides (default: the config's own, BE for C4, RKL2 otherwise)
SEED = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5, "c5v": 5}


def _workload(name, n):
    from paper_2403_01004_b200 import configs
    kw = {} if n is None else {"n": n}
    if name in ("c3", "c4", "c5"):
        return getattr(configs, name)(host=False, **kw)
    if name == "c5v":
        return configs.c5(host=False, **kw)
    if name == "c2":  # grid only (the oracle ranks build their own slabs)
        from paper_2403_01004_b200 import mesh
        nn = n or (128, 128, 256)
        grid = mesh.build_spherical_grid(configs.r_geometric_ratio(nn[0], 1.0, 2.5, 1.01), nn[1], nn[2])
        return configs.Workload("C2", grid, configs.spherical_bc("dirichlet"), 2000.0, 2)
    raise ValueError(name)


# ------------------------------------------------------------------ GPU leg
def run_gpu(case, out, max_cycles=None, from_cycle=None):
    import bench
    from paper_2403_01004_b200 import device, ptl
    name, n = CASES[case]
    ctx = device.default_context()
    t0 = time.perf_counter()
    prob = bench.Problem(name, ctx, n)
    sc = bench.scheme_for(name, types.SimpleNamespace(scheme=SCHEME.get(case), pc="jacobi"))
    prob.reset()
    from paper_2403_01004_b200 import _lib
    for f, _, _, _ in prob.ops:
        np.save(os.path.join(out, f"{case}_{f}_init.npy"), prob.fields[f].download(layout=_lib.LAYOUT_SOA))
    dts = {f: op.device_op(prob.w.grid, nc, ctx).dt_euler for f, op, nc, _ in prob.ops}
    ctx.sync()
    t1 = time.perf_counter()
    remaining = None
    if max_cycles is None and from_cycle is None:
        reps = prob.step(sc, ptl.PtlConfig())
    else:  # a partial step (the field is advanced in place): cycles [from_cycle, from_cycle + max_cycles)
        from paper_2403_01004_b200 import errors
        prob.reset()
        reps = []
        for f, op, nc, _ in prob.ops:
            if op.kind == "aligned":
                op.freeze(prob.fields[f])

        def cycles(f, op, outer, k):
            try:  # the step may also end within these k cycles (the last one)
                return ptl.cycle_operator(op, sc, prob.fields[f], outer, ptl.PtlConfig(max_cycles=k))[1]
            except errors.CycleCapError as e:
                return e.report

        for f, op, nc, _ in prob.ops:
            outer = prob.outer_dt
            if from_cycle:  # run the first cycles, keep their end state, continue from it
                first = cycles(f, op, outer, from_cycle)
                for e in first.entries:  # the C loop's own bookkeeping
                    outer = 0.0 if e.dt == outer else outer - e.dt
                remaining = outer
                np.save(os.path.join(out, f"{case}_{f}_start.npy"), prob.fields[f].download(layout=_lib.LAYOUT_SOA))
            reps.append(cycles(f, op, outer, max_cycles or 1))
    ctx.sync()
    t2 = time.perf_counter()
    rec = {"case": case, "config": name, "grid": list(prob.dg.global_shape), "outer_dt": prob.outer_dt,
           "dt_euler_min": prob.dtE, "dt_euler": dts, "scheme": sc.kind, "tol": sc.tol,
           "step_s": t2 - t1, "setup_s": t1 - t0, "max_cycles": max_cycles, "from_cycle": from_cycle,
           "remaining_dt": remaining, "ops": []}
    for (f, op, nc, _), rep in zip(prob.ops, reps):
        np.save(os.path.join(out, f"{case}_{f}_final.npy"), prob.fields[f].download(layout=_lib.LAYOUT_SOA))
        rec["ops"].append({"field": f, "kind": op.kind, "ncomp": nc,
                           "cycles": [[e.dt, e.iters] for e in rep.entries]})
    with open(os.path.join(out, f"{case}_gpu.json"), "w") as fh:
        json.dump(rec, fh)
    prob.free()
    print(f"[gpu] {case}: step {t2 - t1:.2f} s, " + ", ".join(
        f"{o['field']}: {len(o['cycles'])} cycles / {sum(c[1] for c in o['cycles'])} iters" for o in rec["ops"]),
        flush=True)
    return rec


def run_fake(case, out):
    """CPU self-check of the oracle leg: the single-domain oracle stands in
    for the GPU leg (same files), so the slab oracle must agree with it."""
    from helpers import oracle_aligned, oracle_scalar, soa
    from oracle import ptl as optl
    from paper_2403_01004_b200 import configs
    name, n = CASES[case]
    w = _workload(name, n)
    seed = SEED[name]
    ops = []
    rho = None
    if name in ("c5", "c5v"):
        rho = np.exp(-10.0 * (np.asarray(w.grid.coords[0]) - 1.0))[:, None, None] * np.ones(tuple(w.grid.shape))
    if name in ("c3", "c4", "c5"):
        T = configs.temperature(w.grid, seed)
        ops.append(("T", oracle_aligned(w.grid, w.bc, configs.dipole_bhat(w.grid, seed), T, rho=rho), T[None]))
    if name in ("c2", "c5", "c5v"):
        ops.append(("v", oracle_scalar(w.grid, w.bc, nu=1.0, rho=rho, ncomp=3, vector_metric=True),
                    soa(configs.harmonic_velocity(w.grid, seed))))
    dts = {f: op.euler_dt() for f, op, _ in ops}
    dtE = min(dts.values())
    kind = SCHEME.get(case) or ("backward_euler" if name == "c4" else "rkl2")
    tol = 1e-9 if name in ("c3", "c4") else 1e-10
    rec = {"case": case, "config": name, "grid": list(w.grid.shape), "outer_dt": w.ratio * dtE, "dt_euler_min": dtE,
           "dt_euler": dts, "scheme": kind, "tol": tol, "step_s": 0.0, "setup_s": 0.0, "ops": []}
    for f, op, u in ops:
        np.save(os.path.join(out, f"{case}_{f}_init.npy"), u)
        u2, rep = optl.cycle_operator(op, optl.OracleScheme(kind, tol=tol), u, w.ratio * dtE, dt_euler=dts[f])
        np.save(os.path.join(out, f"{case}_{f}_final.npy"), u2)
        rec["ops"].append({"field": f, "kind": op.kind, "ncomp": op.ncomp, "cycles": [[r.dt, r.iters] for r in rep]})
    with open(os.path.join(out, f"{case}_gpu.json"), "w") as fh:
        json.dump(rec, fh)


# ------------------------------------------------------------------ oracle leg
def _slab_ops(case, slab, grid, bc):
    """The oracle operators of the config on this rank's extended slab, and
    the extended initial states, generated from the host recipes."""
    from helpers import soa
    from oracle import operators as oops
    from oracle.distributed import SlabOperator
    from oracle.ptl import OracleOperator
    from paper_2403_01004_b200 import configs
    name, _ = CASES[case]
    seed = SEED[name]
    lo, ne = slab.i0 - slab.glo, slab.n + slab.glo + slab.ghi
    out = []  # (field, SlabOperator, extended initial state)

    def sop_of(op):
        s = SlabOperator.__new__(SlabOperator)
        s.slab, s.op = slab, op
        return s

    rho = None
    if name in ("c5", "c5v"):
        rho = np.exp(-10.0 * (np.asarray(grid.coords[0]) - 1.0))[lo:lo + ne][:, None, None] * np.ones(
            (ne,) + tuple(grid.shape[1:]))
    if name in ("c3", "c4", "c5"):
        T = configs.temperature(grid, seed, i0=lo, n0=ne)
        b = soa(configs.dipole_bhat(grid, seed, i0=lo, n0=ne))
        c = oops.aligned_coefficient(T, 1.0, None, 1e-10)
        out.append(("T", sop_of(OracleOperator(slab.geom, "aligned", 1, None, rho, False, b, c, 1.0)), T[None]))
    if name in ("c2", "c5", "c5v"):
        v = soa(configs.harmonic_velocity(grid, seed, i0=lo, n0=ne))
        D = 1.0 if rho is None else np.full(rho.shape, 1.0) * rho
        out.append(("v", sop_of(OracleOperator(slab.geom, "scalar", 3, D, rho, True)), v))
    return out


def _oracle_rank(rank, world, port, case, out, gpu_rec, max_cycles=None):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import torch
    import torch.distributed as dist
    from helpers import oracle_geometry
    from oracle import distributed as od
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        name, n = CASES[case]
        w = _workload(name, n)
        geom = oracle_geometry(w.grid, w.bc)
        slab = od.Slab(geom, rank, world)
        ops = _slab_ops(case, slab, w.grid, w.bc)
        res = {"rank": rank, "i0": slab.i0, "n": slab.n, "inputs_bitwise": True, "ops": []}
        dts = {f: sop.euler_dt() for f, sop, _ in ops}
        dtE = min(dts.values())
        outer = w.ratio * dtE
        res["dt_euler"] = dts
        kind = SCHEME.get(case) or ("backward_euler" if name == "c4" else "rkl2")
        tol = 1e-9 if name in ("c3", "c4") else 1e-10
        t0 = time.perf_counter()
        for f, sop, ext in ops:
            u = slab.interior(ext).copy()
            g0 = np.load(os.path.join(out, f"{case}_{f}_init.npy"), mmap_mode="r")[:, slab.i0:slab.i0 + slab.n]
            res["inputs_bitwise"] &= bool(np.array_equal(u, g0))
            outer_f = outer
            if gpu_rec.get("from_cycle"):  # continue from the GPU's state after the first cycles
                u = np.array(np.load(os.path.join(out, f"{case}_{f}_start.npy"),
                                     mmap_mode="r")[:, slab.i0:slab.i0 + slab.n])
                outer_f = gpu_rec["remaining_dt"]
            u, rep = od.slab_cycle_operator(sop, kind, u, outer_f, dts[f], tol=tol, max_iter=100000,
                                            max_cycles=gpu_rec.get("max_cycles") or
                                            (1 if gpu_rec.get("from_cycle") else None))
            g1 = np.load(os.path.join(out, f"{case}_{f}_final.npy"), mmap_mode="r")[:, slab.i0:slab.i0 + slab.n]
            d = np.asarray(g1) - u
            sums = torch.tensor([float(np.sum(d * d)), float(np.sum(u * u)), float(np.max(np.abs(d)))],
                                dtype=torch.float64)
            dist.all_reduce(sums[:2])
            mx = sums[2:].clone()
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            eq = torch.tensor([1 if np.array_equal(g1, u) else 0], dtype=torch.int64)
            dist.all_reduce(eq, op=dist.ReduceOp.MIN)
            res["ops"].append({"field": f, "cycles": [[r.dt, r.iters] for r in rep], "bitwise": bool(eq.item()),
                               "rel_l2": float(np.sqrt(sums[0].item() / sums[1].item())) if sums[1].item() > 0 else 0.0,
                               "max_abs_diff": float(mx.item())})
        res["oracle_s"] = time.perf_counter() - t0
        ok = torch.tensor([1 if res["inputs_bitwise"] else 0], dtype=torch.int64)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        res["inputs_bitwise"] = bool(ok.item())
        if rank == 0:
            with open(os.path.join(out, f"{case}_oracle.json"), "w") as fh:
                json.dump(res, fh)
    finally:
        dist.destroy_process_group()


def run_oracle(case, out, ranks):
    import multiprocessing as mp
    with open(os.path.join(out, f"{case}_gpu.json")) as fh:
        gpu_rec = json.load(fh)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    ps = [ctx.Process(target=_oracle_rank, args=(r, ranks, port, case, out, gpu_rec)) for r in range(ranks)]
    for p in ps:
        p.start()
    for p in ps:
        p.join()
    if any(p.exitcode != 0 for p in ps):
        raise SystemExit(f"oracle ranks failed: {[p.exitcode for p in ps]}")
    with open(os.path.join(out, f"{case}_oracle.json")) as fh:
        orc = json.load(fh)
    return compare(case, gpu_rec, orc, ranks, time.perf_counter() - t0)


def compare(case, gpu, orc, ranks, wall):
    name = gpu["config"]
    be = gpu["scheme"] == "backward_euler"
    summary = {"case": case, "config": name.upper(), "grid": gpu["grid"], "scheme": gpu["scheme"] + "+PTL",
               "outer_dt_over_dtE": gpu["outer_dt"] / gpu["dt_euler_min"], "oracle_ranks": ranks,
               "oracle_wall_s": round(wall, 1), "gpu_step_s": round(gpu["step_s"], 3),
               "inputs_bitwise": orc["inputs_bitwise"], "max_cycles": gpu.get("max_cycles"),
               "from_cycle": gpu.get("from_cycle"),
               "dt_euler_equal": all(gpu["dt_euler"][f] == orc["dt_euler"][f] for f in gpu["dt_euler"]),
               "ops": []}
    ok = summary["inputs_bitwise"] and summary["dt_euler_equal"]
    for go, oo in zip(gpu["ops"], orc["ops"]):
        gi = [c[1] for c in go["cycles"]]
        oi = [c[1] for c in oo["cycles"]]
        gd = [c[0] for c in go["cycles"]]
        od_ = [c[0] for c in oo["cycles"]]
        e = {"field": go["field"], "kind": go["kind"], "cycles": len(gi), "total_iters": sum(gi),
             "oracle_cycles": len(oi), "oracle_total_iters": sum(oi), "counts_identical": gi == oi,
             "dts_identical": gd == od_,
             "dts_max_rel": max((abs(a - b) / abs(b) for a, b in zip(gd, od_)), default=0.0) if len(gd) == len(od_)
             else None,
             "fields_bitwise": oo["bitwise"], "rel_l2": oo["rel_l2"], "max_abs_diff": oo["max_abs_diff"],
             "per_cycle": [[a, b] for a, b in zip(gi, oi)] if len(gi) <= 40 else None}
        e["pass"] = bool(e["counts_identical"] and (e["rel_l2"] <= 1e-10 if be else (e["fields_bitwise"] and
                                                                                  e["dts_identical"])))
        ok = ok and e["pass"]
        summary["ops"].append(e)
    summary["pass"] = bool(ok)
    return summary


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("leg", choices=["gpu", "oracle", "both", "fake"])
    ap.add_argument("case", choices=list(CASES))
    ap.add_argument("--out", default="/tmp/full_parity")
    ap.add_argument("--ranks", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--max-cycles", type=int, default=None, help="partial step: the first K cycles")
    ap.add_argument("--from-cycle", type=int, default=None,
                    help="partial step: run the first K cycles on the GPU, then compare the next --max-cycles "
                         "(default 1) cycles, the oracle starting from the GPU's state after cycle K")
    ap.add_argument("--json", default=None, help="summary output (default gpurun_out/full_parity_<case>.json)")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    if a.leg in ("gpu", "both"):
        run_gpu(a.case, a.out, a.max_cycles, a.from_cycle)
    if a.leg == "fake":
        run_fake(a.case, a.out)
    if a.leg in ("oracle", "both", "fake"):
        name, n = CASES[a.case]
        w = _workload(name, n)
        ranks = min(a.ranks, w.grid.shape[0])
        s = run_oracle(a.case, a.out, ranks)
        path = a.json or os.path.join(ROOT, "gpurun_out", f"full_parity_{a.case}.json")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "w") as fh:
            json.dump(s, fh, indent=1)
        print(json.dumps({k: v for k, v in s.items() if k != "ops"}), flush=True)
        for e in s["ops"]:
            print("   ", json.dumps({k: v for k, v in e.items() if k != "per_cycle"}), flush=True)


if __name__ == "__main__":
    main()
