"""Small cases that drive every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python scripts/sanitize_cases.py [case ...]

cases: tma (19-point TMA march: F+argmax, fused stages, PCG matvec),
cpasync (the cp.async 19-point march), smarch (7-point march, fused 1+2,
3 components with rho), persist (persistent small-grid cycle loop with its
grid barrier), pcg (scalar + aligned BE+PCG, Jacobi and r-line),
split (multi-rank overlap schedule forced on one rank).  Each case also
checks its result against the oracle so a sanitizer-perturbed schedule that
changes results is caught too."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import oracle_aligned, oracle_scalar, soa  # noqa: E402
from oracle import ptl as optl  # noqa: E402
from paper_2403_01004_b200 import configs, operators, ptl, schemes  # noqa: E402


def _aligned_case(n, kind, ratio):
    w = configs.c3(n=n)
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
    T = operators.Field(w.grid, w.fields["T"])
    op = operators.DiffusionOperator.aligned(cfg, T)
    dtE = op.device_op(w.grid, 1).dt_euler
    sc = schemes.SchemeConfig(kind, tol=1e-9)
    out, rep = ptl.cycle_operator(op, sc, T, ratio * dtE)
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme(kind, tol=1e-9), soa(w.fields["T"][..., None]),
                                   ratio * dtE, dt_euler=dtE)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo], (kind, n)
    a, b = out.values[..., 0], uo[0]
    if kind == "backward_euler":
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-10
    else:
        assert np.array_equal(a, b), (kind, n)
    print(f"  aligned {kind} {n}: {rep.n_cycles} cycles {rep.total_iters} iters ok", flush=True)


def case_tma():
    # n2 % 32 == 0 -> TMA staging; 20 theta rows = a ragged theta tile
    _aligned_case((12, 20, 64), "rkl2", 300)
    _aligned_case((12, 20, 64), "backward_euler", 300)


def case_cpasync():
    _aligned_case((10, 12, 48), "rkl2", 200)


def case_smarch():
    w = configs.c2(n=(20, 12, 64))
    rho = np.exp(-2.0 * (np.asarray(w.grid.coords[0]) - 1.0))[:, None, None] * np.ones(tuple(w.grid.shape))
    os.environ["PC_NO_PERSIST"] = "1"  # the marching kernels, not the persistent loop
    try:
        cfg = operators.ScalarDiffusionConfig(nu=1.0, rho=operators.Field(w.grid, rho[..., None]), bc=w.bc,
                                              vector_metric=True)
        op = operators.DiffusionOperator.scalar(cfg, 3)
        v = operators.Field(w.grid, w.fields["v"])
        dtE = op.device_op(w.grid, 3).dt_euler
        out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), v, 400 * dtE)
    finally:
        del os.environ["PC_NO_PERSIST"]
    oop = oracle_scalar(w.grid, w.bc, nu=1.0, rho=rho, ncomp=3, vector_metric=True)
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(w.fields["v"]), 400 * dtE, dt_euler=dtE)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    assert np.array_equal(soa(out.values), uo)
    print(f"  smarch viscous: {rep.n_cycles} cycles {rep.total_iters} stages ok", flush=True)


def case_persist():
    w = configs.c1(n=(12, 12, 24))
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc)
    op = operators.DiffusionOperator.scalar(cfg, 1)
    u = operators.Field(w.grid, w.fields["u"][..., None])
    dtE = op.device_op(w.grid, 1).dt_euler
    for kind in ("rkl2", "rkg2"):
        out, rep = ptl.cycle_operator(op, schemes.SchemeConfig(kind), u, 500 * dtE)
        oop = oracle_scalar(w.grid, w.bc)
        uo, repo = optl.cycle_operator(oop, optl.OracleScheme(kind), soa(w.fields["u"][..., None]), 500 * dtE,
                                       dt_euler=dtE)
        assert [e.iters for e in rep.entries] == [r.iters for r in repo]
        assert np.array_equal(out.values[..., 0], uo[0])
        print(f"  persist {kind}: {rep.n_cycles} cycles ok", flush=True)


def case_pcg():
    w = configs.c1(n=(12, 12, 24))
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc)
    op = operators.DiffusionOperator.scalar(cfg, 1)
    u = operators.Field(w.grid, w.fields["u"][..., None])
    dtE = op.device_op(w.grid, 1).dt_euler
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("backward_euler", tol=1e-10), u, 500 * dtE)
    print(f"  scalar BE: {rep.n_cycles} cycles {rep.total_iters} iterations", flush=True)
    w = configs.c3(n=(12, 20, 64))
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
    T = operators.Field(w.grid, w.fields["T"])
    op = operators.DiffusionOperator.aligned(cfg, T)
    dtE = op.device_op(w.grid, 1).dt_euler
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("backward_euler", tol=1e-9, preconditioner="line-r"),
                                  T, 300 * dtE)
    print(f"  aligned BE line-r: {rep.n_cycles} cycles {rep.total_iters} iterations", flush=True)


def case_split():
    os.environ["PC_SPLIT_STAGE"] = "1"
    try:
        _aligned_case((12, 20, 64), "rkl2", 300)
    finally:
        del os.environ["PC_SPLIT_STAGE"]


CASES = {"tma": case_tma, "cpasync": case_cpasync, "smarch": case_smarch, "persist": case_persist,
         "pcg": case_pcg, "split": case_split}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        print(f"case {nm}", flush=True)
        CASES[nm]()
    print("all cases ok", flush=True)
