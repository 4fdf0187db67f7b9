"""The CPU oracle against every known-answer example the SPEC gives for the
path (SPEC.md §8c list in SURVEY.md), in the Cartesian metric mode."""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import operators as ops
from oracle import ptl as optl
from oracle import schemes as sch
from oracle.geometry import build_geometry


def g1d(n, kind="dirichlet", h=1.0):
    x = np.arange(n) * h
    return build_geometry([x], [(kind, kind)])


def u1(vals):
    return np.asarray(vals, float)[None, :, None, None]


# ---------------------------------------------------------------- operators
def test_scalar_3point_kat():
    """u=[0,0,1,0], dirichlet(0), dx=1 -> F = [0, 1, -2, 0]."""
    F = ops.scalar_apply(g1d(4), u1([0, 0, 1, 0]))
    assert np.array_equal(F.ravel(), [0.0, 1.0, -2.0, 0.0])


def test_scalar_linear_and_constant_give_zero():
    """SPEC.md:113, :115."""
    g = g1d(6)
    assert np.all(ops.scalar_apply(g, u1(np.arange(6.0)))[0, 1:-1] == 0.0)
    assert np.all(ops.scalar_apply(g, u1(np.full(6, 3.5))) == 0.0)


def test_aligned_kat_prefactor_one():
    """b = x, T0 = 1, T = [1,1,2,1] dirichlet(1), prefactor 1 -> interior [1, -2]."""
    g = g1d(4)
    b = np.zeros((3,) + g.shape)
    b[0] = 1.0
    c = ops.aligned_coefficient(np.ones(g.shape))
    F = ops.aligned_apply(g, np.array([1.0, 1, 2, 1])[:, None, None], b, c, pref=1.0)
    assert np.array_equal(F.ravel(), [0.0, 1.0, -2.0, 0.0])


def test_aligned_perpendicular_gradient_vanishes():
    """b = x, T varying only in y -> |F| <= 1e-12 scale."""
    x = np.linspace(0, 1, 7)
    g = build_geometry([x, x], [("neumann", "neumann"), ("neumann", "neumann")])
    b = np.zeros((3,) + g.shape)
    b[0] = 1.0
    T = (1.0 + np.sin(3 * x))[None, :, None] * np.ones(g.shape)
    F = ops.aligned_apply(g, T, b, ops.aligned_coefficient(np.full(g.shape, 2.0)))
    assert np.max(np.abs(F)) <= 1e-12 * np.max(np.abs(T))


def test_aligned_linear_in_x_gives_zero():
    """SPEC.md:123."""
    x = np.linspace(0, 1, 6)
    g = build_geometry([x, x], [("dirichlet", "dirichlet"), ("neumann", "neumann")])
    b = np.zeros((3,) + g.shape)
    b[0] = 1.0
    T = (2.0 + 3.0 * x)[:, None, None] * np.ones(g.shape)
    F = ops.aligned_apply(g, T, b, ops.aligned_coefficient(np.ones(g.shape)))
    assert np.max(np.abs(F[1:-1])) <= 1e-12


def test_aligned_1d_equals_scalar():
    """1-D aligned with b = x reproduces scalar diffusion (1e-14)."""
    rng = np.random.default_rng(0)
    x = np.cumsum(rng.uniform(0.5, 1.5, 9))
    g = build_geometry([x], [("neumann", "dirichlet")])
    c = rng.uniform(0.5, 2.0, g.shape)
    b = np.zeros((3,) + g.shape)
    b[0] = 1.0
    T = rng.normal(size=g.shape)
    Fa = ops.aligned_apply(g, T, b, c)
    Fs = ops.scalar_apply(g, T[None], D=c)[0]
    assert np.max(np.abs(Fa - Fs)) <= 1e-14 * np.max(np.abs(Fs))


def test_aligned_domain_error():
    with pytest.raises(ValueError):
        ops.aligned_coefficient(np.array([1.0, 0.0, 2.0]))


# ---------------------------------------------------------------- dt_Euler
def test_euler_dt_kats():
    """1-D periodic dx^2/2, 2-D h^2/4, nu=0 -> +inf."""
    h = 0.1
    gp = build_geometry([np.arange(10) * h], [("periodic", "periodic")])
    assert math.isclose(ops.euler_dt(ops.scalar_gershgorin(gp)), h * h / 2, rel_tol=1e-14)
    g2 = build_geometry([np.arange(10) * h] * 2, [("periodic", "periodic")] * 2)
    assert math.isclose(ops.euler_dt(ops.scalar_gershgorin(g2)), h * h / 4, rel_tol=1e-14)
    assert ops.euler_dt(ops.scalar_gershgorin(gp, D=0.0)) == math.inf


def test_euler_dt_vs_power_iteration():
    """Gershgorin dt <= the true stable step 2/rho(J) and within 4x."""
    x = np.linspace(0, 1, 9)
    g = build_geometry([x, x], [("neumann", "neumann"), ("dirichlet", "dirichlet")])
    n = int(np.prod(g.shape))
    J = np.zeros((n, n))
    for q in range(n):
        e = np.zeros(n)
        e[q] = 1
        J[:, q] = ops.scalar_apply(g, e.reshape((1,) + g.shape)).ravel()
    free = ~g.pinned.ravel()
    lam = np.max(np.abs(np.linalg.eigvals(J[np.ix_(free, free)])))
    dt = ops.euler_dt(ops.scalar_gershgorin(g))
    assert dt <= 2 / lam * (1 + 1e-12) and dt >= 0.5 / lam


# ---------------------------------------------------------------- PTL
def test_ptl_kat():
    """limited(1/3) at k=2; SPEC.md:381 clamp to dtE = 1/2."""
    g = g1d(4)
    u = u1([0, 0, 1, 0])
    F = ops.scalar_apply(g, u)
    assert optl.compute_ptl(u, F, g) == pytest.approx(1 / 3, rel=0, abs=0)
    assert optl.compute_ptl(u, F, g, check_all=True) <= 1 / 3
    dtE = ops.euler_dt(ops.scalar_gershgorin(g))
    assert dtE == 0.5
    assert max(1 / 3, dtE) == 0.5


def test_ptl_unlimited_cases():
    """constant / linear u -> unlimited -> one cycle."""
    g = g1d(6)
    for u in (u1(np.full(6, 2.0)), u1(np.arange(6.0))):
        F = ops.scalar_apply(g, u)
        F[:, 0] = F[:, -1] = 0.0
        assert optl.compute_ptl(u, F, g) is None
    op = optl.OracleOperator(g, "scalar")
    out, rep = optl.cycle_operator(op, optl.OracleScheme("rkg2"), u1(np.arange(6.0)), 3.0)
    assert len(rep) == 1 and rep[0].dt == 3.0


def test_ptl_argmax_tie_lowest_index():
    """ties in |F| resolve to the lowest linear index (F[1] = F[4] = -2)."""
    g = g1d(7, "dirichlet")
    u = u1([0, 1, 0, 0, 1, 0, 0])
    F = ops.scalar_apply(g, u)
    c, pt, flat = optl._aos_argmax(np.abs(F))
    assert pt == (1, 0, 0)


# ---------------------------------------------------------------- schemes
def test_rkg2_counts_kat():
    """s(1) = 3, s(500) = 55, s(->0) = 3."""
    assert sch.rkg2_iteration_count(1.0, 1.0) == 3
    assert sch.rkg2_iteration_count(500.0, 1.0) == 55
    assert sch.rkg2_iteration_count(1e-9, 1.0) == 3


def test_rkl2_counts():
    assert sch.rkl2_iteration_count(1.0, 1.0) == 2
    assert sch.rkl2_iteration_count(500.0, 1.0) == 45
    assert sch.rkl2_iteration_count(2000.0, 1.0) == 89
    assert sch.rkl2_iteration_count(1e4, 1.0) == 200
    assert sch.rkl2_iteration_count(5e4, 1.0) == 447


def test_rkg2_coefficient_kats():
    """SPEC.md:266-268 and acceptance 10 (Appendix A identities to 1e-14, odd s <= 201)."""
    mu, nu, mut, gam = sch.rkg2_coefficients(5)
    assert math.isclose(mut[1], 1 / 6, rel_tol=1e-15)  # w(5) = 1/6
    assert mu[2] == 0.5 and nu[2] == -0.1 and gam[2] == 0.0
    assert math.isclose(mu[3], 49 / 27, rel_tol=1e-14)
    for s in range(3, 202, 2):
        mu, nu, mut, gam = sch.rkg2_coefficients(s)
        w = Fraction(6, (s + 4) * (s - 1))
        b = [Fraction(1), Fraction(1, 3), Fraction(1, 15)] + [
            Fraction(4 * (k - 1) * (k + 4), 3 * k * (k + 1) * (k + 2) * (k + 3)) for k in range(3, s + 1)]
        assert b[3] == Fraction(7, 135) if s >= 3 else True
        for k in range(3, s + 1):
            muk = (2 + Fraction(1, k)) * b[k] / b[k - 1]
            nuk = -(Fraction(1, k) + 1) * b[k] / b[k - 2]
            gk = (Fraction(k * (k + 1), 2) * b[k - 1] - 1) * muk * w
            assert abs(mu[k] - float(muk)) <= 1e-14 * abs(float(muk))
            assert abs(nu[k] - float(nuk)) <= 1e-14 * abs(float(nuk))
            assert abs(mut[k] - float(muk * w)) <= 1e-14 * abs(float(muk * w))
            assert abs(gam[k] - float(gk)) <= 1e-14 * max(abs(float(gk)), 1e-300)


def _scalar_decay(kind, z, s=None):
    """Run the scheme on u' = -u with dt = -z (a 1-node problem)."""
    class Op:
        def __call__(self, u):
            return -u
    u0 = np.ones((1, 1, 1, 1))
    pinned = np.zeros((1, 1, 1), bool)
    dt = -z
    if kind in ("rkl2", "rkg2"):
        return sch.sts_step(lambda u: -u, u0, -u0, dt, s, kind, pinned)[0, 0, 0, 0]
    raise ValueError


def test_sts_identity_and_accuracy():
    """F = 0 -> identity; du/dt = -u, dt = 1e-3 -> error <= 1e-9."""
    u0 = np.full((1, 3, 1, 1), 2.5)
    pinned = np.zeros((3, 1, 1), bool)
    for kind, s in (("rkl2", 4), ("rkg2", 5)):
        assert np.array_equal(sch.sts_step(lambda u: 0 * u, u0, 0 * u0, 0.1, s, kind, pinned), u0)
        assert abs(_scalar_decay(kind, -1e-3, s) - math.exp(-1e-3)) <= 1e-9


def test_sts_second_order_and_stability():
    """R(0)=1, R'(0)=1, R''(0)=1 and |R| <= 1 on the design interval."""
    for kind, s in (("rkl2", 9), ("rkg2", 9)):
        h = 1e-3
        Rp, R0, Rm = (_scalar_decay(kind, z, s) for z in (h, 0.0, -h))
        assert abs(R0 - 1.0) <= 1e-14  # mu + nu + kap = 1 up to rounding
        assert abs((Rp - Rm) / (2 * h) - 1.0) < 1e-6  # central difference: O(h^2) truncation
        assert abs((Rp - 2 * R0 + Rm) / (h * h) - 1.0) < 1e-3
        zmax = -(s * s + s - 2) / 2 if kind == "rkl2" else -(s + 4) * (s - 1) / 3
        for z in np.linspace(zmax, 0, 400):
            assert abs(_scalar_decay(kind, z, s)) <= 1 + 1e-12


def test_be_amplification_kat():
    """lambda dt = 1000 -> 1/1001."""
    g = g1d(1, "neumann")
    A = lambda x: x + 1000.0 * x
    b = np.ones((1, 1, 1, 1))
    x, it, rel, conv = sch.pcg_solve(A, b, lambda r: r / 1001.0, b, np.ones_like(b), 1e-12, 10)
    assert conv and abs(x.ravel()[0] - 1 / 1001) < 1e-15


def test_pcg_kats():
    """A = I -> 1 iteration; diag(1,2,3) x = (1,2,3) -> x = 1 in 1 iteration."""
    b = np.array([1.0, 2.0, 3.0])[None, :, None, None]
    W = np.ones_like(b)
    x, it, rel, conv = sch.pcg_solve(lambda v: v, b, lambda r: r, np.zeros_like(b), W, 1e-10, 10)
    assert it == 1 and conv and np.array_equal(x, b)
    d = np.array([1.0, 2.0, 3.0])[None, :, None, None]
    x, it, rel, conv = sch.pcg_solve(lambda v: d * v, b, lambda r: r / d, np.zeros_like(b), W, 1e-10, 10)
    assert it == 1 and conv and np.allclose(x, 1.0)


def test_be_pcg_matches_dense_solve():
    """1-D BE (I + alpha L), alpha = 10, n = 64, tol 1e-10 -> dense solve to 1e-8."""
    g = g1d(64, "dirichlet")
    op = optl.OracleOperator(g, "scalar")
    rng = np.random.default_rng(1)
    u = rng.normal(size=(1,) + g.shape)
    u[:, 0] = u[:, -1] = 0.0
    _, dg = op.bound_and_diag()
    x, it, rel, conv = sch.backward_euler_step(op.apply, dg, op.weights(), u, 10.0, 1e-10, 1000, g.pinned)
    n = 64
    J = np.zeros((n, n))
    for q in range(n):
        e = np.zeros((1,) + g.shape)
        e.ravel()[q] = 1
        J[:, q] = op.apply(e).ravel()
    xd = np.linalg.solve(np.eye(n) - 10.0 * J, u.ravel())
    assert conv and np.max(np.abs(x.ravel() - xd)) <= 1e-8 * np.max(np.abs(xd))
    # Jacobi of (I + alpha L), alpha = 1, dx = 1 -> diagonal 3
    assert np.all((1.0 + 1.0 * dg[0, 1:-1]) == 3.0)


def test_be_identity_for_zero_operator():
    """F = 0 -> u^{n+1} = u^n, 1 PCG iteration."""
    g = g1d(5, "neumann")
    op = optl.OracleOperator(g, "scalar", D=0.0)
    u = np.arange(5.0)[None, :, None, None]
    _, dg = op.bound_and_diag()
    x, it, rel, conv = sch.backward_euler_step(op.apply, dg, op.weights(), u, 1.0, 1e-10, 10, g.pinned)
    assert it == 1 and conv and np.array_equal(x, u)


def test_cycle_report_sums_to_outer_dt():
    """sum dt == outer_dt; with the Euler floor n_cycles <= ceil(T/dtE)."""
    g = g1d(32, "dirichlet")
    op = optl.OracleOperator(g, "scalar")
    u = np.zeros((1,) + g.shape)
    u[0, 10:20] = 1.0
    dtE = op.euler_dt()
    T = 50 * dtE
    for kind in ("rkl2", "rkg2", "backward_euler"):
        out, rep = optl.cycle_operator(op, optl.OracleScheme(kind), u, T)
        assert abs(sum(r.dt for r in rep) - T) <= 1e-12 * T
        assert len(rep) <= math.ceil(T / dtE)
        assert all(r.dt >= dtE or r is rep[-1] for r in rep)
