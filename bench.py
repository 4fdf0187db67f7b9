#!/usr/bin/env python
"""Benchmark of the PTL-cycled parabolic advance (BASELINE.json metric:
cell-updates/s per full parabolic step, fp64, with the HBM roofline fraction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]
                    [--decomp r|phi] [--weak] [--scheme rkl2|rkg2|be] [--pc jacobi|line-r] [--no-ptl]

A "step" is one full MAS parabolic step of the chosen config: refresh the
lagged T0 (coefficients + Gershgorin bound) and advance the outer step with
PTL cycling (RKL2 stages or BE+PCG iterations).  Every step starts from the
same seeded initial state (restored by a device copy inside the step), so each
timed step is the same workload.  One cell-update = one cell advanced by one
RKL2 stage or one PCG iteration.  ``--gpus N`` without a
launcher starts the N ranks itself (one per GPU, rendezvous on 127.0.0.1).

  value        = cells x (sum of stages / PCG iterations) / device time of the
                 K steps (CUDA events on the library stream, max over ranks)
  e2e          = the same metric through the public API (ptl.split_advance on
                 host Fields): pinned host -> device copies of the step inputs
                 (T, b, rho, v) and the device -> host copy of the result inside
  roofline     = algorithmic bytes of the dominant hot loop / its device time
                 (CUDA events around its launches), vs the measured HBM copy
                 bandwidth in MEASURED_PEAKS.json; traffic from the committed
                 ncu capture (profiles/ncu_summary.json)
  cpu_baseline = the numpy oracle (oracle/, the "port" of the reference
                 algorithm), 1 host process: per-piece timings of bounded
                 r-chunk samples EXTRAPOLATED to the full step with its exact
                 cycle / stage mix (see STEP_COUNTS)

``--impl reference`` times the same extrapolated oracle on all host cores
(one process per core over r-chunks; the reference repository ships no
implementation of this path) and prints the same metric and config.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# algorithmic bytes per cell-update of the fused stage / PCG iteration
BYTES = {
    ("aligned", "rkl2"): 64,   # reads u_{k-1}, beta(3), u_{k-2}, u0, y0; writes u_k
    ("aligned_rho", "rkl2"): 64,   # + rho, radial (C5: rho(r), read once per plane, not per node)
    ("aligned", "be"): 128,    # Kp: r, p_old, d -> p; K7: p, beta(3) -> Ap; K8: x, r, p, Ap, d -> x, r
    # one rank, point Jacobi: the p-update fused into the matvec march (EpiMatvecP)
    # r, p_old, d, beta(3) -> p, Ap; K8: x, r, p, Ap, d -> x, r
    ("aligned", "be-fused"): 120,
    # r-line preconditioner: z, p_old -> p; p, beta(3) -> Ap; x, r, p, Ap -> x, r;
    # line solve r, jl, inv -> z' and z', cp, r -> z
    ("aligned", "be-line"): 176,
    ("scalar", "rkl2"): 40,    # reads u_{k-1}, u_{k-2}, u0, y0; writes u_k
    ("scalar", "be"): 96,      # K7: r, p, d -> p, Ap;  K8: x, r, p, Ap, d -> x, r
    ("vector", "rkl2"): 120,   # 3 components x 40
    ("vector_rho", "rkl2"): 128,   # + rho (D = nu rho formed per node; a radial rho is read per plane: 120)
}
# the fused stage-1+2 launch of the 7-point march, per cell-update (two per
# launch and cell): reads u0, y0 (+ rho); writes u2 (f12) and u1 (f12w)
BYTES_F12 = {
    ("scalar", "f12"): 12, ("scalar", "f12w"): 16,
    ("vector", "f12"): 36, ("vector", "f12w"): 48,
    ("vector_rho", "f12"): 40, ("vector_rho", "f12w"): 52,
    # the aligned TMA march (EpiStageA12): reads u0, y0, beta(3); writes u2 (+ u1); rho radial (per plane)
    ("aligned", "af12"): 24, ("aligned", "af12w"): 28,
    ("aligned_rho", "af12"): 24, ("aligned_rho", "af12w"): 28,
}

CONFIG_MODEL = {
    "c1": "C1 scalar diffusion 48x48x96 spherical, dt=500 dtE",
    "c2": "C2 vector viscosity 128x128x256x3 spherical, dt=2000 dtE",
    "c3": "C3 Spitzer conduction 256x256x512 spherical, dt=1e4 dtE",
    "c4": "C4 Spitzer conduction 512x512x1024 spherical, BE+PCG tol 1e-9, dt=1e4 dtE",
    "c5": "C5 coupled Spitzer conduction + vector viscosity (rho field) 768x768x1536 spherical, "
          "one split MAS step of 5e4 dtE",
}
CONFIG_MODEL["c5v"] = ("C5 viscosity operator alone (3-component vector viscosity with metric terms, rho field) "
                       "768x768x1536 spherical, one step of 5e4 dtE(viscosity) -- the C5 vector kernel at full weight")
DEFAULT_CONFIG = "c5"
CONFIG_SHAPE = {"c1": (48, 48, 96), "c2": (128, 128, 256), "c3": (256, 256, 512), "c4": (512, 512, 1024),
                "c5": (768, 768, 1536), "c5v": (768, 768, 1536)}


def _vmarch_applies(prob, args):
    """k_vec_march's conditions (capi_ops.cuh vmarch_ok): a spherical grid (phi periodic, theta
    not), phi in whole 32-column tiles, not phi-slabs, PC_NO_VMARCH unset."""
    n2 = int(prob.dg.global_shape[2])
    return (getattr(prob.w.grid, "metric", "") == "spherical" and n2 % 32 == 0
            and getattr(args, "decomp", None) != "phi" and os.environ.get("PC_NO_VMARCH") != "1")


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.limit")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons, under, pw, plim = [], [], set(), [], [], []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                s, m, p = float(f[0]), float(f[1]), float(f[2])
            except ValueError:
                continue
            sm.append(s)
            mx.append(m)
            if p > 300:
                under.append(s)
                pw.append(p)
            try:
                plim.append(float(f[8]))
            except (IndexError, ValueError):
                pass
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        use = under or sm
        return {"sm_mhz": statistics.median(use) if use else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "samples_under_load": len(under),
                "power_w": statistics.median(pw) if pw else None, "power_limit_w": max(plim) if plim else None}


# ---------------------------------------------------------------- workloads

def scheme_for(name, args):
    from paper_2403_01004_b200 import schemes
    if args.scheme:
        kind = {"be": "backward_euler"}.get(args.scheme, args.scheme)
    else:
        kind = "backward_euler" if name == "c4" else "rkl2"
    tol = 1e-9 if name in ("c3", "c4") else 1e-10
    return schemes.SchemeConfig(kind, tol=tol, max_iter=100000, preconditioner=args.pc)


class Problem:
    """The device-resident state of one config: fields, operators and the
    (name, op, kind) list split_advance cycles over.  Inputs of C3-C5 are
    generated in HBM by the library (configs.gen_*, bit-identical to the host
    recipes); C1/C2 are uploaded from the host recipe."""

    def __init__(self, name, ctx, n=None):
        from paper_2403_01004_b200 import configs, device, operators
        self.name = name
        kw = {} if n is None else {"n": n}
        if name in ("c3", "c4", "c5"):
            w = getattr(configs, name)(host=False, **kw)
        elif name == "c5v":
            w = configs.c5(host=False, **kw)
        else:
            w = getattr(configs, name)(**kw)
        self.w = w
        dg = device.device_grid(w.grid, w.bc, ctx)
        self.dg = dg
        self.fields = {}
        self.ops = []  # (state name, DiffusionOperator, ncomp, bytes key)
        if name in ("c3", "c4", "c5"):
            b = configs.gen_dipole(device.DeviceField(dg, 3), w.grid, w.seed)
            rho = configs.gen_radial(device.DeviceField(dg, 1), w.meta["rho_r"]) if name == "c5" else None
            self.fields["T"] = device.DeviceField(dg, 1)
            cfg = operators.AlignedConductionConfig(b_hat=b, rho=rho, m_p=3.0, k_B=1.0, bc=w.bc)
            self.ops.append(("T", operators.DiffusionOperator.aligned(cfg), 1, "aligned_rho" if rho else "aligned"))
            self.b, self.rho = b, rho
            if name == "c5":
                self.fields["v"] = device.DeviceField(dg, 3)
                vcfg = operators.ScalarDiffusionConfig(nu=1.0, rho=rho, bc=w.bc, vector_metric=True)
                self.ops.append(("v", operators.DiffusionOperator.scalar(vcfg, 3), 3, "vector_rho"))
        elif name == "c5v":
            rho = configs.gen_radial(device.DeviceField(dg, 1), w.meta["rho_r"])
            self.rho = rho
            self.fields["v"] = device.DeviceField(dg, 3)
            vcfg = operators.ScalarDiffusionConfig(nu=1.0, rho=rho, bc=w.bc, vector_metric=True)
            self.ops.append(("v", operators.DiffusionOperator.scalar(vcfg, 3), 3, "vector_rho"))
        elif name == "c2":
            self.v0 = device.DeviceField.from_values(dg, w.fields["v"])
            self.fields["v"] = device.DeviceField(dg, 3)
            cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc, vector_metric=True)
            self.ops.append(("v", operators.DiffusionOperator.scalar(cfg, 3), 3, "vector"))
        else:
            self.u0 = device.DeviceField.from_values(dg, w.fields["u"][..., None])
            self.fields["u"] = device.DeviceField(dg, 1)
            cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc)
            self.ops.append(("u", operators.DiffusionOperator.scalar(cfg, 1), 1, "scalar"))
        self.reset()
        dts = []
        for fname, op, nc, _ in self.ops:
            if op.kind == "aligned":
                op.freeze(self.fields[fname])
            dts.append(op.device_op(w.grid, nc, ctx).dt_euler)
        self.dtE = min(dts)
        self.outer_dt = w.ratio * self.dtE

    def reset(self):
        """Back to the seeded initial state (device generation / device copy)."""
        from paper_2403_01004_b200 import configs
        w = self.w
        if "T" in self.fields:
            configs.gen_temperature(self.fields["T"], w.grid, w.seed)
        if self.name in ("c5", "c5v"):
            configs.gen_harmonic(self.fields["v"], w.grid, w.seed)
        elif self.name == "c2":
            self.fields["v"].copy_from(self.v0)
        elif self.name == "c1":
            self.fields["u"].copy_from(self.u0)

    def step(self, sc, pcfg):
        from paper_2403_01004_b200 import ptl
        self.reset()
        st = ptl.split_advance([(f, op) for f, op, _, _ in self.ops], self.fields, self.outer_dt,
                               [(sc, pcfg)] * len(self.ops))
        return st.reports

    def host_inputs(self):
        """Pinned-host copies of every input of a step (for the e2e leg)."""
        out = {}
        for k, f in list(self.fields.items()) + [("b", getattr(self, "b", None)), ("rho", getattr(self, "rho", None))]:
            if f is None:
                continue
            out[k] = np.ascontiguousarray(f.download())
        if self.name in ("c1", "c2"):  # the initial state (fields may have been advanced)
            out[self.ops[0][0]] = np.ascontiguousarray((self.u0 if self.name == "c1" else self.v0).download())
        else:
            self.reset()
            for k in self.fields:
                out[k] = np.ascontiguousarray(self.fields[k].download())
        return out

    def free(self):
        """Release the device state (operators hold reference cycles with
        their device handles: collect them so HBM is returned now)."""
        import gc
        for f in ("fields", "ops", "b", "rho", "u0", "v0"):
            if hasattr(self, f):
                delattr(self, f)
        gc.collect()


# ---------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    from paper_2403_01004_b200 import device, ptl

    uid = None
    dist = None
    if world > 1:
        import torch.distributed as dist_
        dist = dist_
        dist.init_process_group("gloo")
        obj = [device.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    decomp = args.decomp or ("phi" if args.config == "c4" else "r")
    ctx = device.Context(local_rank, world, rank, uid, axis=2 if decomp == "phi" else 0)
    device.set_default_context(ctx)
    name = args.config
    t_setup = time.perf_counter()
    n_over = None if args.n is None else tuple(int(x) for x in args.n.split(","))
    if args.weak and world > 1:  # weak scaling: the config's grid per rank, stacked along the slab axis
        base = n_over or CONFIG_SHAPE[name]
        n_over = (base[0], base[1], base[2] * world) if decomp == "phi" else (base[0] * world, base[1], base[2])
    prob = Problem(name, ctx, n_over)
    sc = scheme_for(name, args)
    pcfg = ptl.PtlConfig(enabled=not args.no_ptl)
    setup_s = time.perf_counter() - t_setup

    for _ in range(args.warmup):
        prob.step(sc, pcfg)
    if dist:
        dist.barrier()
    ctx.sync()
    ctx.reset_stats()
    ctx.enable_timing(True)
    clk = ClockSampler(local_rank)
    clk.start()
    ctx.mark(0)
    total_cu = 0
    reps = []
    for _ in range(args.steps):
        rr = prob.step(sc, pcfg)
        reps.append(rr)
        for (fname, op, nc, bkey), rep in zip(prob.ops, rr):
            total_cu += prob.dg.ncells * rep.total_iters
    ctx.mark(1)
    ms = ctx.elapsed_ms(0, 1)
    clocks = clk.stop()
    st = ctx.stats()
    kinds = ctx.stats_by_kind()
    ctx.enable_timing(False)
    if dist:
        import torch
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        t = torch.tensor([total_cu], dtype=torch.float64)
        dist.all_reduce(t)
        total_cu = int(t.item())
    value = total_cu / (ms / 1e3)
    kind = "be" if sc.kind == "backward_euler" else "rkl2"
    if kind == "be" and sc.preconditioner == "line-r":
        kind = "be-line"
    fusedp = kind == "be" and world == 1 and os.environ.get("PC_PCG_NO_FUSEP") is None
    # roofline: the hot loop with the largest device time, its algorithmic bytes
    rows = []
    for fname, op, nc, bkey in prob.ops:
        if bkey == "vector_rho" and _vmarch_applies(prob, args) and world == 1 and \
                os.environ.get("PC_NO_RADIAL_RHO") is None:
            # C5 / C5v's rho(r) is radial: the vector march reads rho(i) once per plane (DM 3), no rho stream
            bkey = "vector"
        kk = ("pcg_" if kind.startswith("be") else "sts_") + ("aligned" if op.kind == "aligned" else "scalar")
        d = kinds[kk]
        if d["ms"] > 0:
            bpc = BYTES[(bkey, "be-fused")] if (fusedp and op.kind == "aligned") else BYTES[(bkey, kind)]
            rows.append({"kernel": {"sts_aligned": "k_aligned_tma<EpiStage> (TMA march)",
                                    "sts_scalar": ("k_cycle_small<%d> (persistent cycle loop: F, argmax, stages)" % nc
                                                   if prob.dg.ncells * nc <= (1 << 21) else
                                                   "k_scalar_march<" + str(nc) + " comp, SEpiStage>"),
                                    "pcg_aligned": ("k_pcg_pupdate_z + k_aligned_tma<EpiMatvecT> + k_pcg_update1 + "
                                                    "k_line_solve") if kind == "be-line" else
                                                   ("k_aligned_tma<EpiMatvecP> (p-update fused) + k_pcg_update1"
                                                    if fusedp else
                                                    "k_pcg_pupdate + k_aligned_tma<EpiMatvecT> + k_pcg_update1"),
                                    "pcg_scalar": "k_pcg_matvec + k_pcg_update"}[kk],
                         "ms": d["ms"], "bytes_per_cell_update": bpc,
                         "achieved": bpc * d["cell_updates"] / (d["ms"] / 1e3) / 1e9,
                         "launches": d["launches"], "field": fname})
        if op.kind == "aligned" and not kind.startswith("be"):
            for fk in ("af12", "af12w"):
                d = kinds["sts_" + fk]
                if d["ms"] > 0:
                    bpc = BYTES_F12[(bkey, fk)]
                    rows.append({"kernel": "k_aligned_tma<EpiStageA12> (stages 1+2%s)"
                                           % (", u1 written" if fk == "af12w" else ""),
                                 "ms": d["ms"], "bytes_per_cell_update": bpc, "stages_per_launch": 2,
                                 "achieved": bpc * d["cell_updates"] / (d["ms"] / 1e3) / 1e9,
                                 "launches": d["launches"], "field": fname})
        if op.kind != "aligned" and not kind.startswith("be"):
            for fk in ("f12", "f12w"):
                d = kinds["sts_" + fk]
                if d["ms"] > 0:
                    bpc = BYTES_F12[(bkey, fk)]
                    rows.append({"kernel": "k_scalar_march<%d comp, SEpiStage12> (stages 1+2%s)"
                                           % (nc, ", u1 written" if fk == "f12w" else ""),
                                 "ms": d["ms"], "bytes_per_cell_update": bpc, "stages_per_launch": 2,
                                 "achieved": bpc * d["cell_updates"] / (d["ms"] / 1e3) / 1e9,
                                 "launches": d["launches"], "field": fname})
    for r in rows:  # the 3-component spherical launches run on the vector march (csrc/vmarch.cuh) when it applies
        if r["kernel"].startswith("k_scalar_march<3 comp") and _vmarch_applies(prob, args):
            r["kernel"] = r["kernel"].replace("k_scalar_march<3 comp, ", "k_vec_march<")
    dom = max(rows, key=lambda r: r["ms"]) if rows else None
    peak, peak_src = _peaks()

    ops_info = [(f, op.kind, nc) for f, op, nc, _ in prob.ops]
    e2e = None
    if args.e2e:
        e2e = run_e2e(args, prob, sc, pcfg, ctx, dist)

    line = None
    if rank == 0:
        rep0 = reps[-1]
        cells_global = int(np.prod(prob.dg.global_shape))
        line = {
            "metric": "cell-updates/sec per full parabolic step (fp64)",
            "value": value,
            "unit": "cell-updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": "weak" if (args.weak and world > 1) else "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded recipes, configs.py; generated in HBM bit-identically to the host recipe; "
                    "no public dataset exists)",
            "config": workload_config(
                name, world, prob.dg.global_shape, {f: nc for f, _, nc in ops_info},
                sc.kind + ("(" + sc.preconditioner + ")" if sc.kind == "backward_euler" else "") +
                ("" if args.no_ptl else "+PTL"),
                prob.w.ratio,
                [{"field": f, "kind": kd, "cycles": r.n_cycles, "stages_or_iters": r.total_iters}
                 for (f, kd, _), r in zip(ops_info, rep0)],
                total_cu // max(args.steps, 1), decomp),
            "setup_s": round(setup_s, 2),
            "roofline": None if dom is None else {
                "bound": "hbm",
                "kernel": dom["kernel"],
                "achieved": dom["achieved"],
                "peak": peak,
                "unit": "GB/s",
                "frac": dom["achieved"] / peak,
                "traffic": _traffic(name, kind, dom["field"]),
                "bytes_per_cell_update": dom["bytes_per_cell_update"],
                "algorithmic_bytes_per_launch": dom["bytes_per_cell_update"] * dom.get("stages_per_launch", 1)
                                                * cells_global // world,
                "frac_vs_nominal_8tbs": dom["achieved"] / 8000.0,  # B200 datasheet HBM3e figure
                "peak_source": peak_src,
                "kernel_ms_share": dom["ms"] / ms if ms > 0 else None,
                "all_hot_loops": [{k: v for k, v in r.items() if k != "field"} for r in rows if r.get("launches", 1)],
            },
            "gpu_launches": st["launches"],
            "clocks": clocks,
        }
        if e2e is not None:
            line["e2e"] = e2e
        if args.cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(name, procs=1)
    if dist:
        dist.barrier()
    prob.free()
    ctx.close()
    return line


def _traffic(name, kind, field):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture (profiles/ncu_summary.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        e = d.get(f"{name}_{kind}_{field}")
        return None if e is None else e["dram_bytes_per_launch"]
    except Exception:
        return None


def run_e2e(args, prob, sc, pcfg, ctx, dist):
    """The same metric through the public API with every input on the HOST:
    each step uploads its inputs (state fields, b-hat, rho) from pinned host
    memory, advances with ptl.split_advance and downloads the advanced fields;
    the device-resident problem is freed first.  One GPU: host mesh.Fields
    (global arrays).  N GPUs: each rank holds its r-slab of every input in
    pinned host memory and goes through device.DeviceField.upload/download
    around the same split_advance (a global host array per rank would need
    N x the C5 host footprint)."""
    import gc
    from paper_2403_01004_b200 import device, mesh, operators, ptl

    multi = (dist is not None and ctx.nranks > 1) or os.environ.get("BENCH_E2E_SLABS") == "1"
    host = prob.host_inputs()  # this rank's slab, AoS (n0 local, n1, n2, ncomp)
    w, name = prob.w, prob.name
    ops_desc = [(f, op.kind, nc) for f, op, nc, _ in prob.ops]
    outer_dt = prob.outer_dt
    prob.free()
    state_names = [f for f, _, _ in ops_desc]
    outbuf = {f: np.empty_like(host[f]) for f in state_names} if multi else {}
    for a in list(host.values()) + list(outbuf.values()):
        ctx.pin(a)
    h2d = sum(host[k].nbytes for k in host)
    d2h = sum(host[k].nbytes for k in state_names)
    cells = int(np.prod(w.grid.shape))
    cu = 0
    t0 = None
    # one untimed step first (first-touch of host pages, operator/table caches),
    # then exactly args.steps timed steps
    for it in range(args.steps + (1 if args.warmup > 0 else 0)):
        if t0 is None and (it == 1 or args.warmup == 0):
            ctx.sync()
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            cu = 0
        if multi:
            dg = device.device_grid(w.grid, w.bc, ctx)
            dev = {}
            for k, a in host.items():
                dev[k] = device.DeviceField(dg, a.shape[-1])
                dev[k].upload(a)
            src = dev
        else:
            src = host
        ops = []
        for f, kind, nc in ops_desc:
            if kind == "aligned":
                cfg = operators.AlignedConductionConfig(b_hat=src["b"], rho=src.get("rho"), m_p=3.0, k_B=1.0,
                                                        bc=w.bc)
                ops.append((f, operators.DiffusionOperator.aligned(cfg)))
            else:
                cfg = operators.ScalarDiffusionConfig(nu=1.0, rho=src.get("rho"), bc=w.bc, vector_metric=nc == 3)
                ops.append((f, operators.DiffusionOperator.scalar(cfg, nc)))
        if multi:
            state = {f: dev[f] for f in state_names}
        else:
            state = {f: mesh.Field(w.grid, host[f].reshape(tuple(w.grid.shape) + (-1,))) for f in state_names}
        out = ptl.split_advance(ops, state, outer_dt, [(sc, pcfg)] * len(ops))
        reps = out.reports
        if multi:
            for f in state_names:
                out[f].download(outbuf[f])
        cu += cells * sum(r.total_iters for r in reps)
        del ops, out, state
        if multi:
            del dev, src
        gc.collect()  # operator <-> device-handle cycles: return HBM before the next step
    ctx.sync()
    dt = time.perf_counter() - t0
    if dist:
        import torch
        t = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
        b = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64)
        dist.all_reduce(b)
        h2d, d2h = b[0].item(), b[1].item()
    for a in list(host.values()) + list(outbuf.values()):
        ctx.unpin(a)
    return {"value": cu / dt, "unit": "cell-updates/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * dt / args.steps,
            "path": ("device.DeviceField.upload(pinned host slab) -> ptl.split_advance -> download, per rank"
                     if multi else "ptl.split_advance(host Fields, host b-hat/rho) -> pc_cycle per operator")}


# ---------------------------------------------------------------- CPU oracle
# The reference CPU path is the oracle (the reference repository ships no
# implementation of this path).  A full C3-C5 step of it takes
# hours, so it is timed on bounded r-chunk samples of the same workload and
# EXTRAPOLATED to the step with the step's exact work mix:
#   T_step = sum_ops [ t_setup + cycles * (t_F+argmax+PTL + t_stage1) + (stages - cycles) * t_stage ]
# (BE: stages = PCG iterations, t_stage = one PCG iteration, t_stage1 = the
# PCG start r0 = b - A x0), each t_* per cell measured on the sample and
# scaled by the step's cells.  The per-operator cycle / stage counts are the
# config's own (identical on the oracle and the GPU: full-size parity,
# profiles/r02_full_parity_*.json, BENCH_r01.json for C5).
STEP_COUNTS = {  # config -> [(field, kind, ncomp, cycles, stages or PCG iterations)]
    "c1": [("u", "scalar", 1, 477, 962)],
    "c2": [("v", "vector", 3, 327, 803)],
    "c3": [("T", "aligned", 1, 11, 466)],
    "c4": [("T", "aligned", 1, 6, 576)],
    "c5": [("T", "aligned_rho", 1, 45, 1406), ("v", "vector_rho", 3, 1, 2)],
    "c5v": [("v", "vector_rho", 3, 1601, 4202)],
}


def _chunk_ops(name, lo, nplanes):
    """The config's oracle operators on the r-chunk [lo, lo + nplanes) (its
    own sub-domain with pinned ends) and their initial states."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import oracle_aligned, oracle_scalar, soa
    from paper_2403_01004_b200 import configs, mesh
    n = CONFIG_SHAPE[name]
    if name in ("c3", "c4", "c5", "c5v"):
        full = mesh.build_spherical_grid(configs.r_stretched_c3(n[0]), n[1], n[2])
    elif name == "c2":
        full = mesh.build_spherical_grid(configs.r_geometric_ratio(n[0], 1.0, 2.5, 1.01), n[1], n[2])
    else:
        full = mesh.build_spherical_grid(configs.r_uniform(n[0], 1.0, 2.5), n[1], n[2])
    bc = configs.spherical_bc("dirichlet")
    sub = mesh.Grid((full.coords[0][lo:lo + nplanes], full.coords[1], full.coords[2]), full.metric)
    seed = {"c1": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5, "c5v": 5}[name]
    work = []
    if name == "c5v":
        rho = np.exp(-10.0 * (full.coords[0][lo:lo + nplanes] - 1.0))[:, None, None] * np.ones(sub.shape)
        work.append(("v", (sub, bc, 1.0, rho, 3, True),
                     soa(configs.harmonic_velocity(full, seed, i0=lo, n0=nplanes)), oracle_scalar))
    elif name in ("c3", "c4", "c5"):
        T = configs.temperature(full, seed, i0=lo, n0=nplanes)
        b = configs.dipole_bhat(full, seed, i0=lo, n0=nplanes)
        rho = None
        if name == "c5":
            rho = np.exp(-10.0 * (full.coords[0][lo:lo + nplanes] - 1.0))[:, None, None] * np.ones(sub.shape)
        work.append(("T", (sub, bc, b, T, rho), T[None].copy(), oracle_aligned))
        if name == "c5":
            work.append(("v", (sub, bc, 1.0, rho, 3, True),
                         soa(configs.harmonic_velocity(full, seed, i0=lo, n0=nplanes)), oracle_scalar))
    elif name == "c2":
        work.append(("v", (sub, bc, 1.0, None, 3, True), soa(configs.harmonic_velocity(full, 2, i0=lo, n0=nplanes)),
                     oracle_scalar))
    else:
        work.append(("u", (sub, bc), configs.c1().fields["u"][lo:lo + nplanes][None].copy(), oracle_scalar))
    return work


def _oracle_chunk(job):
    """Per-cell times of every piece of the step on one r-chunk sample:
    setup (coefficients + Gershgorin), F + argmax + PTL pairs, stage 1 and a
    stage k >= 2 (RKL2) or the PCG start and one PCG iteration (BE)."""
    name, lo, nplanes = job
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle import ptl as optl
    from oracle import schemes as osch
    be = name == "c4"
    out = {}
    for field, args, u0, make in _chunk_ops(name, lo, nplanes):
        t = time.perf_counter()
        if make.__name__ == "oracle_aligned":
            sub, bc, b, T, rho = args
            op = make(sub, bc, b, T, rho=rho)  # c = f(T0): the coefficient setup
        else:
            op = make(*args[:2], **dict(zip(("nu", "rho", "ncomp", "vector_metric"), args[2:])))
        lam, diag = op.bound_and_diag()
        dtE = optl.ops.euler_dt(lam)
        t_setup = time.perf_counter() - t
        t = time.perf_counter()
        F = op.apply(u0)
        optl.compute_ptl(u0, F, op.geom)
        t_F = time.perf_counter() - t
        cells = int(np.prod(op.geom.shape))
        if be:
            W = op.weights()
            times = []
            for it in (1, 2):  # PCG start + it iterations (tol unreachable)
                t = time.perf_counter()
                osch.backward_euler_step(op.apply, diag, W, u0, 100 * dtE, 1e-300, it, op.geom.pinned)
                times.append(time.perf_counter() - t)
            t_stage = times[1] - times[0]
            t_stage1 = max(times[0] - t_stage, 0.0)
        else:
            times = []
            for s in (2, 3):
                t = time.perf_counter()
                osch.sts_step(op.apply, u0, F, 10 * dtE, s, "rkl2", op.geom.pinned)
                times.append(time.perf_counter() - t)
            t_stage = times[1] - times[0]
            t_stage1 = max(times[0] - t_stage, 0.0)
        out[field] = {"cells": cells, "setup": t_setup / cells, "F": t_F / cells, "stage1": t_stage1 / cells,
                      "stage": t_stage / cells}
    return out


def cpu_baseline(name, procs=1, planes=None):
    """The oracle on ``procs`` host processes (one r-chunk each, run
    concurrently), extrapolated to one full step of the config."""
    n = CONFIG_SHAPE[name]
    planes = planes or {"c1": 48, "c2": 16, "c3": 8, "c4": 3, "c5": 3, "c5v": 3}[name]
    t0 = time.perf_counter()
    jobs = [(name, (k * planes) % max(1, n[0] - planes + 1), planes) for k in range(procs)]
    if procs == 1:
        res = [_oracle_chunk(jobs[0])]
    else:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_oracle_chunk, jobs)
    wall = time.perf_counter() - t0
    cells = int(np.prod(n))
    t_step = 0.0
    parts = {}
    cu = 0
    for field, kind, nc, cycles, stages in STEP_COUNTS[name]:
        # concurrent chunks: per-cell time of the whole machine = the slowest
        # process's per-cell time / procs (perfect r-slab scaling assumed)
        per = {k: max(r[field][k] for r in res) / procs for k in ("setup", "F", "stage1", "stage")}
        t_op = cells * (per["setup"] + cycles * (per["F"] + per["stage1"]) + (stages - cycles) * per["stage"])
        parts[field] = {"cycles": cycles, "stages_or_iters": stages, "t_op_s": round(t_op, 1),
                        "ns_per_cell": {k: round(v * 1e9, 2) for k, v in per.items()}}
        t_step += t_op
        cu += cells * stages
    return {"value": cu / t_step, "unit": "cell-updates/s", "cores": procs, "kind": "port",
            "extrapolated": True, "ms_per_step_extrapolated": 1e3 * t_step,
            "sample": f"{procs} concurrent process(es), each an r-chunk of {planes} planes of {name.upper()} "
                      f"(numpy oracle, oracle/): coefficient setup + Gershgorin, F + argmax + PTL, stage 1 and "
                      f"stage-k (RKL2) / PCG-start and PCG-iteration times per cell, extrapolated with the step's "
                      f"exact cycle and stage counts; sample wall {wall:.1f} s",
            "parts": parts}


def workload_config(name, world, grid, fields, scheme, ratio, operators, cu_per_step, decomp="r"):
    """The `config` dict of both arms (the driver compares them)."""
    cells = int(np.prod(grid))
    return {
        "workload": CONFIG_MODEL[name],
        "config": name.upper(),
        "grid": list(grid),
        "cells": cells,
        "fields": fields,
        "scheme": scheme,
        "outer_dt_over_dtE": ratio,
        "operators": operators,
        "cell_updates_per_step": cu_per_step,
        "decomposition": f"{decomp}-slabs x{world}" if world > 1 else "single GPU",
        "l2": "inputs larger than L2 (each field %.0f MB > 126 MB)" % (cells * 8 / 1e6)
        if cells * 8 > 126e6 else "fields L2-resident (smaller than 126 MB)",
        "parallelism": f"slab{world}",
    }


def reference_config(name, world, decomp=None):
    ops = STEP_COUNTS[name]
    cells = int(np.prod(CONFIG_SHAPE[name]))
    kind = "backward_euler(jacobi)+PTL" if name == "c4" else "rkl2+PTL"
    return workload_config(name, world, CONFIG_SHAPE[name], {f: nc for f, _, nc, _, _ in ops}, kind,
                           {"c1": 500.0, "c2": 2000.0, "c3": 1e4, "c4": 1e4, "c5": 5e4, "c5v": 5e4}[name],
                           [{"field": f, "kind": "aligned" if k.startswith("aligned") else "scalar", "cycles": c,
                             "stages_or_iters": st} for f, k, _, c, st in ops],
                           sum(cells * st for _, _, _, _, st in ops), decomp or ("phi" if name == "c4" else "r"))


def run_reference(args, rank, world):
    """The reference CPU path (the oracle port) on all host cores: each step
    is one bounded concurrent sample extrapolated to the full step; the
    line's value is the median step, its ms_per_step the extrapolated step
    time of the reference on this host."""
    if rank != 0:
        return None
    procs = os.cpu_count() or 1
    for _ in range(min(args.warmup, 1)):  # (one warm-up sample: page-in and imports; keeps the run to minutes)
        cpu_baseline(args.config, procs=procs)
    vals = [cpu_baseline(args.config, procs=procs) for _ in range(args.steps)]
    v = statistics.median(x["value"] for x in vals)
    cb = dict(vals[-1])
    cb["value"] = v
    return {
        "metric": "cell-updates/sec per full parabolic step (fp64)",
        "value": v,
        "unit": "cell-updates/s",
        "impl": "reference",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": statistics.median(x["ms_per_step_extrapolated"] for x in vals),
        "ms_per_step_kind": "extrapolated full step of the reference CPU path (see cpu_baseline.sample)",
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded recipes, configs.py; no public dataset exists)",
        "config": reference_config(args.config, world, args.decomp),
        "note": "the reference repo ships no implementation of this path; its CPU algorithm is the numpy oracle "
                "(oracle/, the SPEC restatement), run on all host cores over r-chunks and extrapolated",
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def spawn_ranks(n):
    """``--gpus N`` without a launcher: start N copies of this command, one
    per GPU (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* as torchrun sets
    them, rendezvous on 127.0.0.1); rank 0's line is the output."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    rcs = [p.wait() for p in procs]
    return max(rcs, key=abs)


def dry_run(rank, world):
    """The launch check: every rank joins the process group and is counted."""
    ranks = 1
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        ranks = int(t.item())
        dist.destroy_process_group()
    return {"dry_run": True, "n_gpus": world, "ranks_joined": ranks, "rank0_pid": os.getpid()} if rank == 0 else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=["c1", "c2", "c3", "c4", "c5", "c5v"])
    ap.add_argument("--scheme", default=None, choices=[None, "rkl2", "rkg2", "be"])
    ap.add_argument("--pc", default="jacobi", choices=["jacobi", "line-r"],
                    help="BE+PCG preconditioner (default: point Jacobi, the SPEC's PC1)")
    ap.add_argument("--n", default=None, help="override the grid, e.g. 96,96,192 (smoke runs only)")
    ap.add_argument("--weak", action="store_true",
                    help="N > 1: weak scaling, the config's grid per rank stacked in r (default: strong, the "
                         "global grid split into r-slabs)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--decomp", default=None, choices=["r", "phi"],
                    help="N > 1: slab axis (default: phi-slabs for C4, as BASELINE.json names them; r-slabs otherwise)")
    ap.add_argument("--no-ptl", action="store_true",
                    help="one cycle of the whole outer step (no PTL cycling; time-to-solution comparisons)")
    ap.add_argument("--dry-run", action="store_true",
                    help="start the N ranks, check the process group, print one line (no GPU work)")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; refusing to produce a "
                         f"mislabelled line\n")
        sys.exit(2)
    if args.dry_run:
        line = dry_run(rank, world)
    elif args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world, local_rank)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
