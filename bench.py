#!/usr/bin/env python
"""Benchmark of the PTL-cycled parabolic advance (BASELINE.json metric:
cell-updates/s per full parabolic step, fp64, with the HBM roofline fraction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

A "step" is one full MAS parabolic step of the chosen config: refresh the
lagged T0 (coefficients + Gershgorin bound) and advance the outer step with
PTL cycling (RKL2 stages or BE+PCG iterations).  Every step starts from the
same seeded initial state (restored by a device copy inside the step), so each
timed step is the same workload.  One cell-update = one cell advanced by one
RKL2 stage or one PCG iteration.

  value        = cells x (sum of stages / PCG iterations) / device time of the
                 K steps (CUDA events on the library stream, max over ranks)
  e2e          = the same metric through the public API (ptl.split_advance on
                 host Fields): pinned host -> device copies of the step inputs
                 (T, b) and the device -> host copy of the result are inside
  roofline     = algorithmic bytes of the fused stage kernels / their device
                 time (CUDA events around the stage launches), vs the measured
                 HBM copy bandwidth in MEASURED_PEAKS.json
  cpu_baseline = the numpy oracle (oracle/, "port" of the reference algorithm)
                 on a bounded r-chunk sample, 1 host thread

``--impl reference`` times the oracle (the reference CPU algorithm; the
reference repository ships no implementation of this path) on all host cores
(one process per core over r-chunks) and prints the same metric.
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
    ("aligned", "be"): 128,    # Kp: r, p_old, d -> p; K7: p, beta(3) -> Ap; K8: x, r, p, Ap, d -> x, r
    ("scalar", "rkl2"): 40,    # reads u_{k-1}, u_{k-2}, u0, y0; writes u_k
    ("scalar", "be"): 96,      # K7: r, p, d -> p, Ap;  K8: x, r, p, Ap, d -> x, r
    ("vector", "rkl2"): 120,   # 3 components x 40
}

CONFIG_MODEL = {
    "c1": "C1 scalar diffusion 48x48x96 spherical, dt=500 dtE",
    "c2": "C2 vector viscosity 128x128x256x3 spherical, dt=2000 dtE",
    "c3": "C3 Spitzer conduction 256x256x512 spherical, dt=1e4 dtE",
    "c4": "C4 Spitzer conduction 512x512x1024 spherical, BE+PCG tol 1e-9, dt=1e4 dtE",
}


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
         "clocks_event_reasons.sw_power_cap")

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
        sm, mx, reasons, under = [], [], set(), []
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
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        use = under or sm
        return {"sm_mhz": statistics.median(use) if use else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "samples_under_load": len(under)}


# ---------------------------------------------------------------- workloads

def build_workload(name, dg_ctx=None, small=None):
    from paper_2403_01004_b200 import configs
    fn = {"c1": configs.c1, "c2": configs.c2, "c3": configs.c3, "c4": configs.c4}[name]
    return fn() if small is None else fn(n=small)


def make_operator(w, name):
    from paper_2403_01004_b200 import operators
    if name in ("c3", "c4"):
        cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
        return operators.DiffusionOperator.aligned(cfg), "T", "aligned", 1
    if name == "c2":
        cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc, vector_metric=True)
        return operators.DiffusionOperator.scalar(cfg, 3), "v", "vector", 3
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc)
    return operators.DiffusionOperator.scalar(cfg, 1), "u", "scalar", 1


def scheme_for(name, args):
    from paper_2403_01004_b200 import schemes
    if args.scheme:
        kind = {"be": "backward_euler"}.get(args.scheme, args.scheme)
    else:
        kind = "backward_euler" if name == "c4" else "rkl2"
    tol = 1e-9 if name in ("c3", "c4") else 1e-10
    return schemes.SchemeConfig(kind, tol=tol, max_iter=100000)


# ---------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    from paper_2403_01004_b200 import device, ptl, mesh

    uid = None
    dist = None
    if world > 1:
        import torch.distributed as dist_
        dist = dist_
        dist.init_process_group("gloo")
        obj = [device.Context.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = device.Context(local_rank, world, rank, uid)
    device.set_default_context(ctx)
    name = args.config
    w = build_workload(name)
    op, fname, opkind, ncomp = make_operator(w, name)
    sc = scheme_for(name, args)
    init = w.fields[fname]
    init4 = init if init.ndim == 4 else init[..., None]
    dop = op.device_op(w.grid, ncomp, ctx)
    dg = dop.dgrid
    u0 = device.DeviceField.from_values(dg, init4)
    u = device.DeviceField(dg, ncomp)
    if op.kind == "aligned":
        op.freeze(u0)
    dtE0 = dop.dt_euler
    outer_dt = w.ratio * dtE0
    pcfg = ptl.PtlConfig()

    def step():
        u.copy_from(u0)
        if op.kind == "aligned":
            dop.freeze(u)
        _, rep = ptl.cycle_operator(op, sc, u, outer_dt, pcfg)
        return rep

    for _ in range(args.warmup):
        rep = step()
    if dist:
        dist.barrier()
    ctx.sync()
    ctx.reset_stats()
    ctx.enable_timing(True)
    clk = ClockSampler(local_rank)
    clk.start()
    ctx.mark(0)
    total_iters = 0
    reps = []
    for _ in range(args.steps):
        rep = step()
        reps.append(rep)
        total_iters += rep.total_iters
    ctx.mark(1)
    ms = ctx.elapsed_ms(0, 1)
    clocks = clk.stop()
    st = ctx.stats()
    ctx.enable_timing(False)
    if dist:
        import torch
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    cells_global = int(np.prod(dg.global_shape))
    value = cells_global * total_iters / (ms / 1e3)
    kind = "be" if sc.kind == "backward_euler" else "rkl2"
    bpc = BYTES[(opkind, kind)]
    n_stage_cells = dg.ncells * (sum(max(e.iters - 1, 0) for r in reps for e in r.entries) if kind == "rkl2"
                                 else total_iters)
    achieved = bpc * n_stage_cells / (st["stage_ms"] / 1e3) / 1e9 if st["stage_ms"] > 0 else None
    peak, peak_src = _peaks()

    # e2e: the public API with host buffers (rank 0 only at N=1; all ranks otherwise)
    e2e = None
    if args.e2e:
        e2e = run_e2e(args, w, name, op, fname, ncomp, init4, outer_dt, sc, pcfg, ctx, dist)

    line = None
    if rank == 0:
        rep0 = reps[-1]
        line = {
            "metric": "cell-updates/sec per full parabolic step (fp64)",
            "value": value,
            "unit": "cell-updates/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms / args.steps,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (seeded recipe, configs.py; no public dataset exists)",
            "config": {
                "workload": CONFIG_MODEL[name],
                "config": name.upper(),
                "grid": list(dg.global_shape) + ([3] if ncomp == 3 else []),
                "cells": cells_global,
                "scheme": sc.kind + "+PTL",
                "outer_dt_over_dtE": w.ratio,
                "cycles_per_step": rep0.n_cycles,
                "cell_updates_per_step": cells_global * rep0.total_iters,
                "stages_or_iters_per_step": rep0.total_iters,
                "decomposition": f"r-slabs x{world}" if world > 1 else "single GPU",
                "l2": "inputs larger than L2 (each field %.0f MB > 126 MB)" % (cells_global * 8 / 1e6)
                if cells_global * 8 > 126e6 else "fields L2-resident (smaller than 126 MB)",
                "parallelism": f"slab{world}",
            },
            "roofline": {
                "bound": "hbm",
                "kernel": {"aligned": "k_aligned_march<EpiStage>", "scalar": "k_stage<ScalarOp>",
                           "vector": "k_stage<ScalarOp> (3 comp)"}[opkind] if kind == "rkl2"
                else ("k_pcg_pupdate + k_aligned_march<EpiMatvec> + k_pcg_update" if opkind == "aligned"
                      else "k_pcg_matvec + k_pcg_update"),
                "achieved": achieved,
                "peak": peak,
                "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": _traffic(name, kind),
                "bytes_per_cell_update": bpc,
                "peak_source": peak_src,
                "kernel_ms_share": st["stage_ms"] / ms if ms > 0 else None,
            },
            "gpu_launches": st["launches"],
            "clocks": clocks,
        }
        if e2e is not None:
            line["e2e"] = e2e
        if args.cpu_baseline and world >= 1:
            line["cpu_baseline"] = cpu_baseline(name, args.cpu_sample_s)
    if dist:
        dist.barrier()
    ctx.close()
    return line


def _traffic(name, kind):
    """DRAM bytes per cell-update of the stage kernel from the committed ncu
    capture (profiles/ncu_summary.json), or None."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get(f"{name}_{kind}", {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def run_e2e(args, w, name, op, fname, ncomp, init4, outer_dt, sc, pcfg, ctx, dist):
    """The same metric through ptl.split_advance on host Fields (H2D / D2H inside)."""
    from paper_2403_01004_b200 import mesh, operators, ptl

    host_in = np.ascontiguousarray(init4)
    ctx.pin(host_in)
    b_host = None
    if op.kind == "aligned":
        b_host = np.ascontiguousarray(w.fields["b"])
        ctx.pin(b_host)
    h2d = host_in.nbytes + (b_host.nbytes if b_host is not None else 0)
    d2h = host_in.nbytes
    iters = 0
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if op.kind == "aligned":
            cfg = operators.AlignedConductionConfig(b_hat=b_host, m_p=3.0, k_B=1.0, bc=w.bc)
            opx = operators.DiffusionOperator.aligned(cfg)
        else:
            opx = op
        state = {fname: mesh.Field(w.grid, host_in)}
        out, reps = ptl.split_advance([(fname, opx)], state, outer_dt, [(sc, pcfg)])
        iters += sum(r.total_iters for r in reps)
    ctx.sync()
    dt = time.perf_counter() - t0
    if dist:
        import torch
        t = torch.tensor([dt], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    cells = int(np.prod(w.grid.shape))
    ctx.unpin(host_in)
    if b_host is not None:
        ctx.unpin(b_host)
    return {"value": cells * iters / dt, "unit": "cell-updates/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * dt / args.steps,
            "path": "ptl.split_advance(host Field) -> pc_cycle"}


# ---------------------------------------------------------------- CPU oracle

def _oracle_chunk(job):
    """Run `stages` oracle RKL2 stages on an r-chunk (its own sub-domain)."""
    name, lo, nplanes, stages = job
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import oracle_aligned, oracle_scalar, soa
    from oracle import schemes as osch
    from paper_2403_01004_b200 import configs, mesh
    n = {"c1": (48, 48, 96), "c2": (128, 128, 256), "c3": (256, 256, 512), "c4": (512, 512, 1024)}[name]
    if name in ("c3", "c4"):
        full = mesh.build_spherical_grid(configs.r_stretched_c3(n[0]), n[1], n[2])
    elif name == "c2":
        full = mesh.build_spherical_grid(configs.r_geometric_ratio(n[0], 1.0, 2.5, 1.01), n[1], n[2])
    else:
        full = mesh.build_spherical_grid(configs.r_uniform(n[0], 1.0, 2.5), n[1], n[2])
    bc = configs.spherical_bc("dirichlet")
    sub = mesh.Grid((full.coords[0][lo:lo + nplanes], full.coords[1], full.coords[2]), full.metric)
    if name in ("c3", "c4"):
        T = configs.temperature(full, 3, i0=lo, n0=nplanes)
        b = configs.dipole_bhat(full, 3, i0=lo, n0=nplanes)
        op = oracle_aligned(sub, bc, b, T)
        u0 = T[None].copy()
    elif name == "c2":
        op = oracle_scalar(sub, bc, ncomp=3, vector_metric=True)
        u0 = soa(configs.harmonic_velocity(full, 2, i0=lo, n0=nplanes))
    else:
        op = oracle_scalar(sub, bc)
        u0 = configs.c1().fields["u"][lo:lo + nplanes][None].copy()
    dtE = op.euler_dt()
    y0 = op.apply(u0)
    t = time.perf_counter()
    osch.sts_step(op.apply, u0, y0, 10 * dtE, stages, "rkl2", op.geom.pinned)
    dt = time.perf_counter() - t
    return int(np.prod(op.geom.shape)) * (stages - 1), dt  # stages 2..s each one full pass


def cpu_baseline(name, budget_s=20.0, procs=1):
    """Oracle (numpy, single thread) on an r-chunk sample."""
    n0 = {"c1": 48, "c2": 128, "c3": 256, "c4": 512}[name]
    planes = {"c1": 48, "c2": 16, "c3": 8, "c4": 4}[name]
    stages = 4
    t0 = time.perf_counter()
    jobs = [(name, (k * planes) % (n0 - planes), planes, stages) for k in range(procs)]
    if procs == 1:
        res = [_oracle_chunk(jobs[0])]
    else:
        import multiprocessing as mp
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_oracle_chunk, jobs)
    cells = sum(r[0] for r in res)
    secs = max(r[1] for r in res)
    return {"value": cells / secs, "unit": "cell-updates/s", "cores": procs, "kind": "port",
            "sample": f"{procs} x r-chunk of {planes} planes of {name.upper()}, {stages - 1} fused RKL2 stages each "
                      f"(numpy oracle, oracle/operators.py); wall {time.perf_counter() - t0:.1f} s"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    procs = os.cpu_count() or 1
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(args.config, procs=procs)
    t_all = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(args.config, procs=procs))
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
        "ms_per_step": 1e3 * (time.perf_counter() - t_all) / max(args.steps, 1),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded recipe, configs.py)",
        "config": {"workload": CONFIG_MODEL[args.config], "config": args.config.upper(),
                   "note": "the reference repo ships no implementation of this path; its CPU algorithm is "
                           "the numpy oracle (oracle/), run on all host cores over r-chunks"},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "cell-updates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--scheme", default=None, choices=[None, "rkl2", "rkg2", "be"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-cpu-baseline", dest="cpu_baseline", action="store_false")
    ap.add_argument("--cpu-sample-s", type=float, default=20.0)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world, local_rank)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
