"""The SPEC's known-answer examples run through the PRODUCT path on the GPU
(public API -> C ABI -> sm_100a kernels, Cartesian metric mode), the SPEC's
error contracts raised by the device path, and edge-case grids.

Golden values are the SPEC's own (SPEC.md line cited per test; the same cases
pin the oracle in tests/test_oracle_kat.py).  Error cases are checked against
the oracle's decision (which stage blows up, how many cycles fit under the
cap)."""
import math

import numpy as np
import pytest

from helpers import oracle_aligned, oracle_scalar, soa
from oracle import ptl as optl
from oracle import schemes as osch
from paper_2403_01004_b200 import configs, errors, linsolve, mesh, operators, ptl, schemes

pytestmark = pytest.mark.gpu


def grid1d(n, h=1.0):
    return mesh.build_grid([n], coords=[np.arange(n) * h])


def field1d(grid, vals):
    return mesh.Field(grid, np.asarray(vals, float).reshape(grid.shape + (1,)))


# ---------------------------------------------------------------- operators
def test_scalar_3point_kat_on_gpu(gpu_ctx):
    """u = [0,0,1,0], dirichlet(0), dx = 1 -> F = [0, 1, -2, 0]."""
    g = grid1d(4)
    bc = mesh.BoundaryCondition.dirichlet(0.0, 1)
    F = operators.apply_scalar_diffusion(field1d(g, [0, 0, 1, 0]), operators.ScalarDiffusionConfig(nu=1.0, bc=bc))
    assert np.array_equal(F.values.ravel(), [0.0, 1.0, -2.0, 0.0])


def test_scalar_linear_and_constant_on_gpu(gpu_ctx):
    """linear u -> 0 in the interior, constant u -> 0."""
    g = grid1d(6)
    bc = mesh.BoundaryCondition.dirichlet(0.0, 1)
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=bc)
    assert np.all(operators.apply_scalar_diffusion(field1d(g, np.arange(6.0)), cfg).values.ravel()[1:-1] == 0.0)
    bcn = mesh.BoundaryCondition.neumann(1)
    cfgn = operators.ScalarDiffusionConfig(nu=1.0, bc=bcn)
    assert np.all(operators.apply_scalar_diffusion(field1d(g, np.full(6, 3.5)), cfgn).values == 0.0)


def test_aligned_kat_on_gpu(gpu_ctx):
    """b = x, T0 = 1, T = [1,1,2,1] dirichlet(1), prefactor 1 -> interior [1, -2]."""
    g = grid1d(4)
    bc = mesh.BoundaryCondition.dirichlet(1.0, 1)
    b = np.zeros(g.shape + (3,))
    b[..., 0] = 1.0
    cfg = operators.AlignedConductionConfig(b_hat=b, m_p=3.0, k_B=1.0, bc=bc)  # (5/3 - 1) * 3 / 2 = 1
    F = operators.apply_aligned_conduction(field1d(g, [1, 1, 2, 1]), cfg, field1d(g, np.ones(4)))
    assert np.array_equal(F.values.ravel(), [0.0, 1.0, -2.0, 0.0])


def test_aligned_domain_error_on_gpu(gpu_ctx):
    """a non-positive T0 is a domain error."""
    g = grid1d(4)
    bc = mesh.BoundaryCondition.dirichlet(1.0, 1)
    b = np.zeros(g.shape + (3,))
    b[..., 0] = 1.0
    cfg = operators.AlignedConductionConfig(b_hat=b, bc=bc)
    with pytest.raises(errors.DomainError):
        operators.apply_aligned_conduction(field1d(g, [1, 1, 2, 1]), cfg, field1d(g, [1.0, 0.0, 2.0, 1.0]))


# ---------------------------------------------------------------- dt_Euler
def test_euler_dt_kats_on_gpu(gpu_ctx):
    """1-D periodic dx^2/2, 2-D h^2/4, nu = 0 -> +inf."""
    h = 0.1
    g1 = mesh.build_grid([10], coords=[np.arange(10) * h])
    p1 = mesh.BoundaryCondition.periodic(1)
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=p1), 1)
    dt1 = operators.estimate_euler_dt(op, mesh.Field.full(g1, 0.0))
    assert math.isclose(dt1, h * h / 2, rel_tol=1e-14)
    g2 = mesh.build_grid([10, 10], coords=[np.arange(10) * h] * 2)
    p2 = mesh.BoundaryCondition.periodic(2)
    op2 = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=p2), 1)
    assert math.isclose(operators.estimate_euler_dt(op2, mesh.Field.full(g2, 0.0)), h * h / 4, rel_tol=1e-14)
    op0 = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=0.0, bc=p1), 1)
    assert operators.estimate_euler_dt(op0, mesh.Field.full(g1, 0.0)) == math.inf


# ---------------------------------------------------------------- PTL
def test_ptl_kat_on_gpu(gpu_ctx):
    """u = [0,0,1,0] -> k = 2, pairs 1/3 and 1/2 -> limited(1/3);
    SPEC.md:381: the cycle clamps it to dt_E = 1/2."""
    g = grid1d(4)
    bc = mesh.BoundaryCondition.dirichlet(0.0, 1)
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=bc)
    u = field1d(g, [0, 0, 1, 0])
    F = operators.apply_scalar_diffusion(u, cfg)
    lim = ptl.compute_ptl(u, F, g, bc=bc)
    assert float(lim) == 1.0 / 3.0
    op = operators.DiffusionOperator.scalar(cfg, 1)
    dtE = operators.estimate_euler_dt(op, u)
    assert dtE == 0.5
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), u, 2.0)
    assert rep.entries[0].dt == 0.5 and rep.entries[0].limited


def test_ptl_unlimited_one_cycle_on_gpu(gpu_ctx):
    """F = 0 everywhere -> unlimited -> one cycle of the whole step."""
    g = grid1d(6)
    bc = mesh.BoundaryCondition.dirichlet(0.0, 1)
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=bc), 1)
    u = field1d(g, np.zeros(6))
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkg2"), u, 3.0)
    assert rep.n_cycles == 1 and rep.entries[0].dt == 3.0 and not rep.entries[0].limited


# ---------------------------------------------------------------- PCG / BE
def test_pcg_kats_on_gpu(gpu_ctx):
    """A = I -> 1 iteration; diag(1,2,3) x = (1,2,3) -> x = (1,1,1) in 1 iteration."""
    g = mesh.build_grid([3], coords=[np.arange(3.0)])
    bc = mesh.BoundaryCondition.neumann(1)
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=0.0, bc=bc), 1)
    b = field1d(g, [1.0, 2.0, 3.0])
    A = linsolve.LinearOperatorAction(op, 1.0)
    x, st = linsolve.pcg_solve(A, b, linsolve.build_jacobi(A, g), field1d(g, np.zeros(3)), 1e-10, 10)
    assert st.iterations == 1 and st.converged and np.array_equal(x.values.ravel(), [1.0, 2.0, 3.0])
    A2 = linsolve.LinearOperatorAction(op, 1.0, a=np.array([1.0, 2.0, 3.0]))
    x2, st2 = linsolve.pcg_solve(A2, b, linsolve.build_jacobi(A2, g), field1d(g, np.zeros(3)), 1e-10, 10)
    assert st2.iterations == 1 and st2.converged and np.allclose(x2.values.ravel(), 1.0, rtol=0, atol=1e-15)


def test_be_pcg_matches_dense_solve_on_gpu(gpu_ctx):
    """1-D BE (I + alpha L), alpha = 10, n = 64, tol 1e-10 -> dense solve to 1e-8;
    SPEC.md:199: Jacobi diagonal of (I + L), dx = 1 -> 3."""
    n = 64
    g = grid1d(n)
    bc = mesh.BoundaryCondition.dirichlet(0.0, 1)
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=bc), 1)
    rng = np.random.default_rng(1)
    u = rng.normal(size=n)
    u[0] = u[-1] = 0.0
    x, st = schemes.step_backward_euler(op, field1d(g, u), 10.0, schemes.SchemeConfig("backward_euler", tol=1e-10))
    J = np.zeros((n, n))
    for q in range(n):
        e = np.zeros(n)
        e[q] = 1.0
        J[:, q] = op.apply(field1d(g, e)).values.ravel()
    xd = np.linalg.solve(np.eye(n) - 10.0 * J, u)
    assert st.converged and np.max(np.abs(x.values.ravel() - xd)) <= 1e-8 * np.max(np.abs(xd))
    d = op.device_op(g, 1).diagonal().download().ravel()
    assert np.all((1.0 + d[1:-1]) == 3.0)


def test_be_identity_for_zero_operator_on_gpu(gpu_ctx):
    """F = 0 -> u^{n+1} = u^n after 1 PCG iteration."""
    g = grid1d(5)
    bc = mesh.BoundaryCondition.neumann(1)
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=0.0, bc=bc), 1)
    u = field1d(g, np.arange(5.0))
    x, st = schemes.step_backward_euler(op, u, 1.0, schemes.SchemeConfig("backward_euler", tol=1e-10))
    assert st.iterations == 1 and st.converged and np.array_equal(x.values, u.values)


def test_sts_identity_for_zero_operator_on_gpu(gpu_ctx):
    """F = 0 -> the STS step is the identity (both schemes) up to
    the rounding of mu a + nu a + (1 - mu - nu) a (a few ulp), and bitwise the
    oracle's recurrence."""
    g = grid1d(7)
    bc = mesh.BoundaryCondition.neumann(1)
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=0.0, bc=bc), 1)
    vals = np.linspace(1.0, 2.0, 7)
    pinned = np.zeros((7, 1, 1), bool)
    for step, kind in ((schemes.step_rkl2, "rkl2"), (schemes.step_rkg2, "rkg2")):
        out = step(op, field1d(g, vals), 0.3, 0.01).values.ravel()
        s = (osch.rkl2_iteration_count if kind == "rkl2" else osch.rkg2_iteration_count)(0.3, 0.01)
        u0 = vals[None, :, None, None]
        ref = osch.sts_step(lambda u: 0.0 * u, u0, 0.0 * u0, 0.3, s, kind, pinned).ravel()
        assert np.array_equal(out, ref)
        assert np.max(np.abs(out - vals)) <= 32 * np.finfo(float).eps * 2.0


# ---------------------------------------------------------------- error contracts
def test_blowup_names_the_oracle_stage(gpu_ctx):
    """a non-finite stage raises, naming the stage -- the same
    stage the oracle names.  An understated dt_Euler (dt_E given = 150 x the
    true bound) makes the 3-stage step unstable, so a large spike overflows a
    few stages in."""
    w = configs.c1(n=(12, 12, 24))
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc)
    op = operators.DiffusionOperator.scalar(cfg, 1)
    oop = oracle_scalar(w.grid, w.bc)
    dtE = oop.euler_dt()
    dt, dt_given = 300 * dtE, 150 * dtE
    s = osch.rkl2_iteration_count(dt, dt_given)
    found = None
    for e in range(200, 309):
        u = w.fields["u"].copy()
        u[6, 6, 12] = 10.0 ** e
        try:
            osch.sts_step(oop.apply, soa(u[..., None]), oop.apply(soa(u[..., None])), dt, s, "rkl2",
                          oop.geom.pinned)
        except osch.BlowUpError as ex:
            if ex.stage >= 2:
                found = (u, ex.stage)
                break
    assert found is not None, "no oracle blow-up after stage 1 in the scanned amplitudes"
    u, stage = found
    with pytest.raises(errors.BlowUpError) as ei:
        schemes.step_rkl2(op, mesh.Field(w.grid, u[..., None]), dt, dt_given)
    assert ei.value.stage == stage


def test_cycle_cap_returns_partial_report(gpu_ctx):
    """max_cycles exceeded -> error carrying the partial report
    (the same first cycles as the oracle)."""
    w = configs.c1(n=(12, 12, 24))
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc)
    op = operators.DiffusionOperator.scalar(cfg, 1)
    oop = oracle_scalar(w.grid, w.bc)
    dtE = oop.euler_dt()
    u = mesh.Field(w.grid, w.fields["u"][..., None])
    with pytest.raises(errors.CycleCapError) as ei:
        ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), u, 500 * dtE, ptl.PtlConfig(max_cycles=3))
    rep = ei.value.report
    with pytest.raises(optl.CycleCapError) as eo:
        optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(w.fields["u"][..., None]), 500 * dtE,
                            max_cycles=3, dt_euler=dtE)
    orep = eo.value.report
    assert rep.n_cycles == 3
    assert [e.dt for e in rep.entries] == [r.dt for r in orep]
    assert [e.iters for e in rep.entries] == [r.iters for r in orep]


def test_indefinite_system_raises(gpu_ctx):
    """(I + dt J) with dt < 0 large is indefinite -> the
    Jacobi build (non-positive diagonal) refuses it."""
    g = grid1d(16)
    bc = mesh.BoundaryCondition.dirichlet(0.0, 1)
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=bc), 1)
    A = linsolve.LinearOperatorAction(op, -10.0)
    with pytest.raises(errors.IndefiniteOperatorError):
        linsolve.build_jacobi(A, g)


# ---------------------------------------------------------------- edge-case grids
@pytest.mark.parametrize("n", [(3, 3, 4), (3, 5, 32), (5, 17, 33), (4, 33, 64), (7, 3, 96)],
                         ids=["min", "one-tile", "ragged-phi", "ragged-theta-tma", "two-rows"])
def test_edge_grids_aligned_parity(gpu_ctx, n):
    """Minimum sizes, ragged theta and phi tiles, a single tile, TMA and
    cp.async staging: apply, Gershgorin and a PTL-cycled RKL2 step, bitwise."""
    w = configs.c3(n=n)
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
    T = operators.Field(w.grid, w.fields["T"])
    op = operators.DiffusionOperator.aligned(cfg, T)
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
    assert np.array_equal(op.apply(T).values[..., 0], oop.apply(soa(w.fields["T"][..., None]))[0])
    dtE = op.device_op(w.grid, 1).dt_euler
    assert dtE == oop.euler_dt()
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), T, 50 * dtE)
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(w.fields["T"][..., None]), 50 * dtE,
                                   dt_euler=dtE)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    assert np.array_equal(out.values[..., 0], uo[0])


@pytest.mark.parametrize("n", [(3, 3, 4), (5, 9, 40)], ids=["min", "ragged"])
def test_edge_grids_viscous_parity(gpu_ctx, n):
    w = configs.c2(n=n)
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc, vector_metric=True)
    op = operators.DiffusionOperator.scalar(cfg, 3)
    v = operators.Field(w.grid, w.fields["v"])
    oop = oracle_scalar(w.grid, w.bc, ncomp=3, vector_metric=True)
    assert np.array_equal(np.moveaxis(op.apply(v).values, -1, 0), oop.apply(soa(w.fields["v"])))
    dtE = op.device_op(w.grid, 3).dt_euler
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), v, 20 * dtE)
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(w.fields["v"]), 20 * dtE, dt_euler=dtE)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    assert np.array_equal(np.moveaxis(out.values, -1, 0), uo)


def test_cycle_blowup_is_reported_with_the_oracle_stage(gpu_ctx):
    """pc_cycle checks the non-finite flag one cycle late (no per-step host
    sync): the error still names the oracle's stage."""
    w = configs.c1(n=(12, 12, 24))
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc)
    op = operators.DiffusionOperator.scalar(cfg, 1)
    oop = oracle_scalar(w.grid, w.bc)
    dtE = oop.euler_dt()
    u = w.fields["u"].copy()
    u[6, 6, 12] = 1e305
    with pytest.raises(optl.sch.BlowUpError) as eo:
        optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(u[..., None]), 300 * dtE, use_ptl=False,
                            dt_euler=150 * dtE)
    with pytest.raises(errors.BlowUpError) as ei:
        ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), mesh.Field(w.grid, u[..., None]), 300 * dtE,
                           ptl.PtlConfig(enabled=False), dt_euler=150 * dtE)
    assert ei.value.stage == eo.value.stage


# ---------------------------------------------------------------- domain checks on the device
def test_field_count_matches_numpy(gpu_ctx):
    """pc_field_count (the device-side domain test behind the constructors'
    rho validation) counts exactly what numpy counts, NaN failing every test."""
    from paper_2403_01004_b200 import _lib, device

    w = configs.c2(n=(12, 10, 20))
    rng = np.random.default_rng(7)
    v = rng.standard_normal(tuple(w.grid.shape) + (3,))
    v.flat[rng.choice(v.size, 9, replace=False)] = 0.0
    v.flat[rng.choice(v.size, 4, replace=False)] = np.nan
    v.flat[rng.choice(v.size, 3, replace=False)] = np.inf
    v.flat[rng.choice(v.size, 2, replace=False)] = -np.inf
    dg = device.device_grid(w.grid, w.bc)
    f = device.DeviceField.from_values(dg, v)
    with np.errstate(invalid="ignore"):
        want = {_lib.TEST_POSITIVE: int(np.sum(~(v > 0))), _lib.TEST_NONNEG: int(np.sum(~(v >= 0))),
                _lib.TEST_FINITE: int(np.sum(~np.isfinite(v)))}
    for t, n in want.items():
        assert f.count_failing(t) == n, t


@pytest.mark.parametrize("bad", [0.0, -1e-300, np.nan])
@pytest.mark.parametrize("kind", ["scalar", "aligned"])
def test_rho_validation_on_device(gpu_ctx, kind, bad):
    """a density with any !(rho > 0) node raises ValueError at
    operator construction (checked on the device after the upload)."""
    w = configs.c3(n=(8, 8, 16))
    rho = np.full(tuple(w.grid.shape), 2.0)
    if kind == "scalar":
        mk = lambda r: operators.DiffusionOperator.scalar(  # noqa: E731
            operators.ScalarDiffusionConfig(nu=1.0, rho=r, bc=w.bc), 1).device_op(w.grid, 1)
    else:
        mk = lambda r: operators.DiffusionOperator.aligned(  # noqa: E731
            operators.AlignedConductionConfig(b_hat=w.fields["b"], rho=r, m_p=3.0, k_B=1.0, bc=w.bc),
            operators.Field(w.grid, w.fields["T"])).device_op(w.grid, 1)
    mk(rho)  # valid
    rho[3, 5, 7] = bad
    with pytest.raises(ValueError, match="rho must be > 0"):
        mk(rho)
