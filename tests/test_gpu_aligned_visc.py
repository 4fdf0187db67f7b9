"""Parity of the 19-point aligned (Spitzer) and the vector-viscosity paths
(C3 / C4 / C2 recipes at reduced size) against the CPU oracle."""
import numpy as np
import pytest

from helpers import oracle_aligned, oracle_scalar, soa
from oracle import ptl as optl
from paper_2403_01004_b200 import configs, operators, ptl, schemes

pytestmark = pytest.mark.gpu


# (24, 24, 48): cp.async staging (n2 % 32 != 0); (20, 40, 64): TMA bulk-tensor
# staging with partial theta tiles (zero-filled out-of-range rows)
@pytest.fixture(scope="module", params=[(24, 24, 48), (20, 40, 64)], ids=["cpasync", "tma"])
def c3s(request):
    return configs.c3(n=request.param)


def _aligned(w):
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
    return operators.DiffusionOperator.aligned(cfg, operators.Field(w.grid, w.fields["T"]))


def test_aligned_apply_and_bound_bitwise(gpu_ctx, c3s):
    op = _aligned(c3s)
    T = operators.Field(c3s.grid, c3s.fields["T"])
    F = op.apply(T)
    oop = oracle_aligned(c3s.grid, c3s.bc, c3s.fields["b"], c3s.fields["T"])
    Fo = oop.apply(soa(c3s.fields["T"][..., None]))
    assert np.array_equal(F.values[..., 0], Fo[0])
    assert op.device_op(c3s.grid, 1).dt_euler == oop.euler_dt()
    d = op.device_op(c3s.grid, 1).diagonal().download()[..., 0]
    assert np.array_equal(d, oop.bound_and_diag()[1][0])


def test_aligned_rkl2_ptl_parity(gpu_ctx, c3s):
    op = _aligned(c3s)
    dtE = op.device_op(c3s.grid, 1).dt_euler
    T = operators.Field(c3s.grid, c3s.fields["T"])
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), T, 1e4 * dtE)
    oop = oracle_aligned(c3s.grid, c3s.bc, c3s.fields["b"], c3s.fields["T"])
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(c3s.fields["T"][..., None]), 1e4 * dtE,
                                   dt_euler=dtE)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    assert [e.dt for e in rep.entries] == [r.dt for r in repo]
    assert np.array_equal(out.values[..., 0], uo[0])


def test_aligned_be_pcg_parity(gpu_ctx, c3s):
    op = _aligned(c3s)
    dtE = op.device_op(c3s.grid, 1).dt_euler
    T = operators.Field(c3s.grid, c3s.fields["T"])
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("backward_euler", tol=1e-9), T, 1e4 * dtE)
    oop = oracle_aligned(c3s.grid, c3s.bc, c3s.fields["b"], c3s.fields["T"])
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("backward_euler", tol=1e-9),
                                   soa(c3s.fields["T"][..., None]), 1e4 * dtE, dt_euler=dtE)
    assert len(rep.entries) == len(repo)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    a, b = out.values[..., 0], uo[0]
    assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-10


@pytest.mark.parametrize("pc", ["jacobi", "line-r"])
@pytest.mark.parametrize("rho", [False, True])
def test_aligned_be_128bit_pcg_kernels(gpu_ctx, c3s, monkeypatch, pc, rho):
    """The 128-bit p-update / x,r-update kernels (n2 even, the default) and
    the 64-bit ones (PC_PCG_SCALAR_IO): same iteration counts, fields within
    the PCG tolerance contract (the partial sums take nodes in another order),
    both against the oracle."""
    w = c3s
    assert w.grid.shape[2] % 2 == 0
    rr = np.exp(-2.0 * (np.asarray(w.grid.coords[0]) - 1.0))
    rho_a = np.broadcast_to(rr[:, None, None], tuple(w.grid.shape)) * (
        1.0 + 0.05 * np.random.default_rng(3).random(tuple(w.grid.shape))) if rho else None
    T = operators.Field(w.grid, w.fields["T"])
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("PC_PCG_SCALAR_IO", env)
        cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], rho=rho_a, m_p=3.0, k_B=1.0, bc=w.bc)
        op = operators.DiffusionOperator.aligned(cfg, T)
        dtE = op.device_op(w.grid, 1).dt_euler
        o, rep = ptl.cycle_operator(op, schemes.SchemeConfig("backward_euler", tol=1e-9, preconditioner=pc), T,
                                    1e4 * dtE)
        outs.append((o.values[..., 0].copy(), [e.iters for e in rep.entries]))
    assert outs[0][1] == outs[1][1]
    a, b = outs
    assert np.linalg.norm(a[0] - b[0]) / np.linalg.norm(b[0]) <= 1e-12
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"], rho=rho_a)
    sch = optl.OracleScheme("backward_euler", tol=1e-9)
    if pc == "line-r":
        sch.preconditioner = "line-r"
    uo, repo = optl.cycle_operator(oop, sch, soa(w.fields["T"][..., None]), 1e4 * dtE, dt_euler=dtE)
    assert a[1] == [r.iters for r in repo]
    assert np.linalg.norm(a[0] - uo[0]) / np.linalg.norm(uo[0]) <= 1e-10


@pytest.fixture(scope="module")
def c2s():
    return configs.c2(n=(20, 24, 48))


def test_viscous_rkl2_ptl_parity(gpu_ctx, c2s):
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=c2s.bc, vector_metric=True)
    op = operators.DiffusionOperator.scalar(cfg, 3)
    v = operators.Field(c2s.grid, c2s.fields["v"])
    F = op.apply(v)
    oop = oracle_scalar(c2s.grid, c2s.bc, ncomp=3, vector_metric=True)
    Fo = oop.apply(soa(c2s.fields["v"]))
    assert np.array_equal(np.moveaxis(F.values, -1, 0), Fo)
    dtE = op.device_op(c2s.grid, 3).dt_euler
    assert dtE == oop.euler_dt()
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), v, 2000 * dtE)
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(c2s.fields["v"]), 2000 * dtE, dt_euler=dtE)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    assert [e.dt for e in rep.entries] == [r.dt for r in repo]
    assert np.array_equal(np.moveaxis(out.values, -1, 0), uo)


def test_tma_and_cpasync_paths_bitwise(gpu_ctx, monkeypatch):
    """The TMA-staged and the cp.async-staged marching kernels give identical bits."""
    import os
    w = configs.c3(n=(16, 40, 64))
    T = operators.Field(w.grid, w.fields["T"])
    out = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("PC_NO_TMA", env)
        op = _aligned(w)
        dtE = op.device_op(w.grid, 1).dt_euler
        o, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), T, 300 * dtE)
        out.append((o.values.copy(), [e.iters for e in rep.entries]))
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0], out[1][0])


@pytest.mark.parametrize("kind,n,no_tma", [("aligned", (24, 40, 64), False), ("aligned", (24, 24, 48), True),
                                           ("viscous", (40, 24, 64), False)],
                         ids=["aligned-tma", "aligned-cpasync", "viscous"])
def test_split_stage_launches_bitwise(gpu_ctx, monkeypatch, kind, n, no_tma):
    """The multi-rank overlap schedule (interior r-chunks launched while the
    halo planes travel, then the two boundary chunks) forced on one rank
    (PC_SPLIT_STAGE): bitwise the single-launch stages, same counts."""
    if no_tma:
        monkeypatch.setenv("PC_NO_TMA", "1")
    if kind == "aligned":
        w = configs.c3(n=n)
        T = operators.Field(w.grid, w.fields["T"])
        make = lambda: _aligned(w)  # noqa: E731
        nc = 1
    else:
        w = configs.c2(n=n)
        T = operators.Field(w.grid, w.fields["v"])
        make = lambda: operators.DiffusionOperator.scalar(  # noqa: E731
            operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc, vector_metric=True), 3)
        nc = 3
    out = []
    for split in (False, True):
        if split:
            monkeypatch.setenv("PC_SPLIT_STAGE", "1")
        op = make()
        dtE = op.device_op(w.grid, nc).dt_euler
        o, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), T, 200 * dtE)
        out.append((o.values.copy(), [e.iters for e in rep.entries]))
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0], out[1][0])


def test_fused_pupdate_matvec_bitwise(gpu_ctx, monkeypatch):
    """EpiMatvecP (the p-update fused into the TMA matvec march: r, p_old, d
    staged, p formed in shared memory) is bitwise the separate p-update
    kernel + matvec: same iteration counts, residuals and field bits."""
    w = configs.c4(n=(24, 40, 64))
    T = operators.Field(w.grid, w.fields["T"])
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("PC_PCG_NO_FUSEP", env)
        else:
            monkeypatch.delenv("PC_PCG_NO_FUSEP", raising=False)
        op = _aligned(w)
        dtE = op.device_op(w.grid, 1).dt_euler
        out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("backward_euler", tol=1e-9), T, 1e4 * dtE)
        outs.append(([e.iters for e in rep.entries], [e.relres for e in rep.entries], out.values.copy()))
    assert sum(outs[0][0]) > 20
    assert outs[0][0] == outs[1][0] and outs[0][1] == outs[1][1]
    assert np.array_equal(outs[0][2], outs[1][2])
