"""SPEC acceptance criteria 4, 5, 6 and 9 through the
PRODUCT path (public API -> C ABI -> sm_100a kernels), each run also checked
against the CPU oracle on the same inputs (cycle counts equal, STS fields
bitwise, BE fields within the PCG contract)."""
import numpy as np
import pytest

from acceptance_cases import (RATIO, STEP_CASES, coords, neighbours, oracle_geom, random_fields, sign_changes,
                              step_values)
from helpers import oracle_scalar, soa
from oracle import ptl as optl
from paper_2403_01004_b200 import configs, mesh, operators, ptl, schemes

pytestmark = pytest.mark.gpu


def _same_dts(a, b, kind):
    """STS fields are bitwise the oracle's, so every PTL (and cycle dt) is
    too; a BE field agrees to the PCG contract (~1e-10), so the PTL of the
    next cycle agrees to about that (the cycle counts stay identical)."""
    if kind == "backward_euler":
        assert len(a) == len(b) and np.allclose(a, b, rtol=1e-8, atol=0.0)
    else:
        assert a == b


def _setup(dim, n):
    g = mesh.build_grid([n] * dim, coords=coords(dim, n))
    bc = mesh.BoundaryCondition.neumann(dim)
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=bc), 1)
    return g, bc, op


def _run(dim, n, kind, use_ptl, static=False):
    g, bc, op = _setup(dim, n)
    dtE = op.device_op(g, 1).dt_euler
    u0 = step_values(dim, n)
    cfg = ptl.PtlConfig(enabled=use_ptl, reevaluate="static" if static else "dynamic")
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig(kind, tol=1e-10), mesh.Field(g, u0[..., None]),
                                  RATIO * dtE, cfg)
    # the oracle on the same input
    og = oracle_geom(dim, n)
    oop = optl.OracleOperator(og, "scalar", 1, 1.0, None, False)
    assert oop.euler_dt() == dtE
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme(kind, tol=1e-10), u0.reshape(og.shape)[None],
                                   RATIO * dtE, use_ptl=use_ptl, static=static)
    a, b = out.values[..., 0], uo[0].reshape((n,) * dim)
    gi, oi = [e.iters for e in rep.entries], [r.iters for r in repo]
    if kind == "backward_euler" and len(repo) > 50:
        # hundreds of chained BE solves (static cycling): each agrees with the
        # oracle to the PCG contract, so a count near the tolerance edge may
        # flip by one iteration; the cycle structure is identical
        assert len(gi) == len(oi) and max(abs(x - y) for x, y in zip(gi, oi)) <= 1
        assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(b)
        return a, rep
    assert gi == oi
    _same_dts([e.dt for e in rep.entries], [r.dt for r in repo], kind)
    if kind == "backward_euler":
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    else:
        assert np.array_equal(a, b)
    return a, rep


@pytest.mark.parametrize("dim,n", STEP_CASES)
def test_acceptance4_on_gpu(gpu_ctx, dim, n):
    init = sign_changes(step_values(dim, n))
    u_free, _ = _run(dim, n, "rkg2", False)
    u_ptl, _ = _run(dim, n, "rkg2", True)
    assert sign_changes(u_free) > init
    assert sign_changes(u_ptl) <= init
    b_free, _ = _run(dim, n, "backward_euler", False)
    b_ptl, _ = _run(dim, n, "backward_euler", True)
    assert sign_changes(b_ptl) <= sign_changes(b_free)


@pytest.mark.parametrize("dim,n", STEP_CASES)
@pytest.mark.parametrize("kind", ["rkg2", "rkl2", "backward_euler"])
def test_acceptance6_static_vs_dynamic_on_gpu(gpu_ctx, dim, n, kind):
    _, dyn = _run(dim, n, kind, True)
    _, sta = _run(dim, n, kind, True, static=True)
    assert dyn.n_cycles <= sta.n_cycles
    if dim == 2:
        assert dyn.n_cycles < sta.n_cycles
    assert len({e.dt for e in sta.entries[:-1]}) == 1
    assert all(e.ptl_raw == sta.entries[0].ptl_raw for e in sta.entries)


def test_acceptance5_on_gpu(gpu_ctx):
    """Eq. 3 after a GPU explicit Euler step at the GPU's limited PTL, at
    every pair adjacent to the |F| maximum, 1000 seeded random fields."""
    limited = 0
    for u in random_fields(1000):
        dim = u.ndim
        g = mesh.build_grid(list(u.shape), coords=[np.linspace(0.0, 1.0, m) for m in u.shape])
        bc = mesh.BoundaryCondition.neumann(dim)
        cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=bc)
        op = operators.DiffusionOperator.scalar(cfg, 1)
        U = mesh.Field(g, u[..., None])
        F = op.apply(U)
        p = ptl.compute_ptl(U, F, g, ptl.PtlConfig(), bc=bc)
        if p is ptl.UNLIMITED:
            continue
        limited += 1
        u1 = schemes.step_euler(op, U, p).values[..., 0]
        absF = np.abs(F.values[..., 0])
        k = np.unravel_index(int(np.argmax(absF)), u.shape)
        scale = float(np.max(np.abs(u))) ** 2
        for nb in neighbours(u.shape, k):
            assert (u1[k] - u1[nb]) * (u[k] - u[nb]) >= -1e-14 * scale
    assert limited >= 900


@pytest.mark.parametrize("kind,ratio", [("euler", 0.5), ("rkl2", 20.0), ("rkg2", 20.0), ("backward_euler", 20.0)])
@pytest.mark.parametrize("use_ptl", [False, True])
def test_acceptance9_conservation_on_gpu(gpu_ctx, kind, ratio, use_ptl):
    """Neumann (zero-flux) diffusion conserves sum(rho V u) to 1e-12 relative
    over 100 outer steps, for the Cartesian 2-D case of the oracle test and a
    spherical shell (Neumann r-ends, axis, periodic phi).  The explicit and
    STS schemes conserve to round-off; a BE step conserves to its PCG
    tolerance (the iterates are not conservative), so the BE leg solves to
    1e-13 to meet the 1e-12 bar over 100 steps."""
    x = np.linspace(0.0, 1.0, 24)
    cases = [(mesh.build_grid([24, 24], coords=[x, x]), mesh.BoundaryCondition.neumann(2)),
             (mesh.build_spherical_grid(np.linspace(1.0, 2.0, 10), 8, 16), configs.spherical_bc("neumann"))]
    for g, bc in cases:
        op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=bc), 1)
        W = oracle_scalar(g, bc).weights()[0].reshape(tuple(g.shape))
        u0 = np.random.default_rng(9).random(tuple(g.shape))
        dt = ratio * op.device_op(g, 1).dt_euler
        u = mesh.Field(g, u0[..., None])
        for _ in range(100):
            u, _ = ptl.cycle_operator(op, schemes.SchemeConfig(kind, tol=1e-13), u, dt,
                                      ptl.PtlConfig(enabled=use_ptl))
        s0, s1 = float(np.sum(W * u0)), float(np.sum(W * u.values[..., 0]))
        assert abs(s1 - s0) <= 1e-12 * abs(s0), (g.metric, s0, s1)


@pytest.mark.parametrize("kind", ["euler", "backward_euler", "rkl2", "rkg2"])
def test_acceptance8_on_gpu(gpu_ctx, kind):
    """Criterion 8 through the GPU path (aligned operator on a 2-D periodic
    Cartesian grid): every dt's final field equals the oracle's (bitwise,
    BE to 1e-10) and the errors against the fine-Euler oracle decrease
    monotonically to below 1e-6."""
    from acceptance_cases import ANISO_STEPS, aniso_problem, aniso_reference
    from oracle import ptl as optl
    dtE_o, ref, oop = aniso_reference()
    x, u0, b = aniso_problem()
    g = mesh.build_grid([len(x), len(x)], coords=[x, x])
    per = mesh.FaceBC("periodic")
    bc = mesh.BoundaryCondition(((per, per), (per, per)))
    cfg = operators.AlignedConductionConfig(b_hat=b, m_p=3.0, k_B=1.0, bc=bc)
    op = operators.DiffusionOperator.aligned(cfg, mesh.Field(g, np.ones(u0.shape + (1,))))
    dtE = op.device_op(g, 1).dt_euler
    assert dtE == dtE_o
    errs = []
    for m in ANISO_STEPS:
        u = mesh.Field(g, u0[..., None])
        uo = u0.reshape((1,) + oop.geom.shape)
        for _ in range(m):
            u, _ = ptl.cycle_operator(op, schemes.SchemeConfig(kind, tol=1e-13), u, dtE / m,
                                      ptl.PtlConfig(enabled=False))
            uo, _ = optl.cycle_operator(oop, optl.OracleScheme(kind, tol=1e-13), uo, dtE / m, use_ptl=False)
        a, o = u.values[..., 0], uo.reshape(u0.shape)
        if kind == "backward_euler":
            assert np.linalg.norm(a - o) <= 1e-10 * np.linalg.norm(o)
        else:
            assert np.array_equal(a, o)
        errs.append(float(np.max(np.abs(a - ref))))
    assert all(q < p for p, q in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-6, errs
