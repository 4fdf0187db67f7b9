"""PtlConfig knobs through the GPU path against the oracle: static
first-PTL cycling and the per-cycle lagged-T0 refresh
(SPEC.md:385), on the C3 recipe at reduced size (both staging paths of the
19-point march) and the C1 recipe (7-point, host-driven loop)."""
import numpy as np
import pytest

from helpers import oracle_aligned, oracle_scalar, soa
from oracle import operators as oops
from oracle import ptl as optl
from paper_2403_01004_b200 import configs, operators, ptl, schemes

pytestmark = pytest.mark.gpu


def _same_dts(a, b, kind):
    """STS fields are bitwise the oracle's, so every PTL (and cycle dt) is
    too; a BE field agrees to the PCG contract (~1e-10), so the PTL of the
    next cycle agrees to about that (the cycle counts stay identical)."""
    if kind == "backward_euler":
        assert len(a) == len(b) and np.allclose(a, b, rtol=1e-8, atol=0.0)
    else:
        assert a == b


@pytest.fixture(scope="module", params=[(24, 24, 48), (20, 40, 64)], ids=["cpasync", "tma"])
def c3s(request):
    return configs.c3(n=request.param)


def _aligned(w):
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
    return operators.DiffusionOperator.aligned(cfg, operators.Field(w.grid, w.fields["T"]))


@pytest.mark.parametrize("kind", ["rkl2", "rkg2", "backward_euler"])
def test_static_ptl_aligned_parity(gpu_ctx, c3s, kind):
    op = _aligned(c3s)
    dtE = op.device_op(c3s.grid, 1).dt_euler
    T = operators.Field(c3s.grid, c3s.fields["T"])
    sc = schemes.SchemeConfig(kind, tol=1e-9)
    out, rep = ptl.cycle_operator(op, sc, T, 300 * dtE, ptl.PtlConfig(reevaluate="static"))
    oop = oracle_aligned(c3s.grid, c3s.bc, c3s.fields["b"], c3s.fields["T"])
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme(kind, tol=1e-9), soa(c3s.fields["T"][..., None]),
                                   300 * dtE, dt_euler=dtE, static=True)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    _same_dts([e.dt for e in rep.entries], [r.dt for r in repo], kind)
    a, b = out.values[..., 0], uo[0]
    if kind == "backward_euler":
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    else:
        assert np.array_equal(a, b)
    # dynamic re-evaluation never needs more cycles
    _, dyn = ptl.cycle_operator(op, sc, T, 300 * dtE)
    assert dyn.n_cycles <= rep.n_cycles


@pytest.mark.parametrize("kind", ["rkl2", "backward_euler"])
def test_per_cycle_T0_refresh_parity(gpu_ctx, c3s, kind):
    """refresh_T0='cycle': the aligned operator is re-frozen at T0 := u at
    the start of every cycle (coefficients, Gershgorin bound, Jacobi
    diagonal); Delta t_E follows the refreshed operator."""
    op = _aligned(c3s)
    dtE0 = op.device_op(c3s.grid, 1).dt_euler
    T = operators.Field(c3s.grid, c3s.fields["T"])
    sc = schemes.SchemeConfig(kind, tol=1e-9)
    # (ratio 100: longer steps undershoot T below 0 on these coarse grids,
    # which a per-cycle refresh rightly reports as a domain error)
    out, rep = ptl.cycle_operator(op, sc, T, 100 * dtE0, ptl.PtlConfig(refresh_T0="cycle"))
    oop = oracle_aligned(c3s.grid, c3s.bc, c3s.fields["b"], c3s.fields["T"])

    def refresh(o, u):
        o.c = oops.aligned_coefficient(u[0], 1.0, None, 1e-10)

    uo, repo = optl.cycle_operator(oop, optl.OracleScheme(kind, tol=1e-9), soa(c3s.fields["T"][..., None]),
                                   100 * dtE0, refresh_cycle=refresh)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    _same_dts([e.dt for e in rep.entries], [r.dt for r in repo], kind)
    a, b = out.values[..., 0], uo[0]
    if kind == "backward_euler":
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    else:
        assert np.array_equal(a, b)
    # the default (once per outer step) is a different advance
    out2, rep2 = ptl.cycle_operator(op.freeze(T), sc, T, 100 * dtE0)
    assert not np.array_equal(out2.values, out.values)


def test_static_ptl_scalar_host_loop(gpu_ctx):
    """Static mode on a small scalar grid runs the host-driven loop (the
    persistent kernel implements dynamic cycling only): bitwise the oracle."""
    w = configs.c1(n=(16, 16, 32))
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc), 1)
    u = operators.Field(w.grid, w.fields["u"][..., None])
    dtE = op.device_op(w.grid, 1).dt_euler
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), u, 500 * dtE, ptl.PtlConfig(reevaluate="static"))
    oop = oracle_scalar(w.grid, w.bc)
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(w.fields["u"][..., None]), 500 * dtE,
                                   dt_euler=dtE, static=True)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    assert np.array_equal(out.values[..., 0], uo[0])


def test_refresh_rejected_for_scalar(gpu_ctx):
    w = configs.c1(n=(8, 8, 16))
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc), 1)
    u = operators.Field(w.grid, w.fields["u"][..., None])
    with pytest.raises(ValueError):
        ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), u, 1e-3, ptl.PtlConfig(refresh_T0="cycle"))
