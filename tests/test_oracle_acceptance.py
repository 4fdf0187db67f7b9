"""SPEC acceptance criteria 4, 5, 6 and 9 on the CPU
oracle (the same criteria run through the GPU path in
test_gpu_acceptance.py)."""
import numpy as np
import pytest

from acceptance_cases import (RATIO, STEP_CASES, neighbours, oracle_geom, random_fields, sign_changes,
                              step_values)
from oracle import operators as ops
from oracle import ptl as optl
from oracle.geometry import build_geometry


def _op(geom):
    return optl.OracleOperator(geom, "scalar", 1, 1.0, None, False)


def _run(dim, n, kind, use_ptl, static=False):
    g = oracle_geom(dim, n)
    op = _op(g)
    dtE = op.euler_dt()
    u0 = step_values(dim, n).reshape(g.shape)[None]
    u, rep = optl.cycle_operator(op, optl.OracleScheme(kind, tol=1e-10), u0, RATIO * dtE, use_ptl=use_ptl,
                                 static=static)
    return u[0].reshape((n,) * dim), rep


@pytest.mark.parametrize("dim,n", STEP_CASES)
def test_acceptance4_ptl_suppresses_oscillations(dim, n):
    """Criterion 4 (§4.1): RKG2 without PTL adds sign changes,
    RKG2 with PTL cycling does not, BE with PTL <= BE without."""
    init = sign_changes(step_values(dim, n))
    u_free, _ = _run(dim, n, "rkg2", False)
    u_ptl, _ = _run(dim, n, "rkg2", True)
    assert sign_changes(u_free) > init
    assert sign_changes(u_ptl) <= init
    b_free, _ = _run(dim, n, "backward_euler", False)
    b_ptl, _ = _run(dim, n, "backward_euler", True)
    assert sign_changes(b_ptl) <= sign_changes(b_free)


@pytest.mark.parametrize("dim,n", STEP_CASES)
def test_acceptance6_dynamic_needs_no_more_cycles_than_static(dim, n):
    """Criterion 6 ("much fewer overall cycles"): dynamic
    re-evaluation <= static first-PTL cycling, strictly fewer in 2-D."""
    _, dyn = _run(dim, n, "rkg2", True)
    _, sta = _run(dim, n, "rkg2", True, static=True)
    assert len(dyn) <= len(sta)
    if dim == 2:
        assert len(dyn) < len(sta)
    # the static mode reuses the first PTL: every cycle but the last is the same dt
    assert len({r.dt for r in sta[:-1]}) == 1


def test_acceptance5_euler_step_at_ptl_keeps_signs():
    """Criterion 5 (Eq. 3): an explicit Euler step at the
    limited PTL keeps the sign of every difference adjacent to the |F|
    maximum, over 1000 seeded random fields."""
    limited = 0
    for u in random_fields(1000):
        g = build_geometry([np.linspace(0.0, 1.0, m) for m in u.shape], [("neumann", "neumann")] * u.ndim)
        U = u.reshape(g.shape)[None]
        F = ops.scalar_apply(g, U)
        ptl = optl.compute_ptl(U, F, g)
        if ptl is None:
            continue
        limited += 1
        u1 = U + ptl * F
        _, k, _ = optl._aos_argmax(np.abs(F))
        scale = float(np.max(np.abs(U))) ** 2
        for nb in neighbours(g.shape, k):
            d0 = float(U[(0,) + k] - U[(0,) + nb])
            d1 = float(u1[(0,) + k] - u1[(0,) + nb])
            assert d1 * d0 >= -1e-14 * scale
    assert limited >= 900


SCHEMES = [("euler", 0.5), ("rkl2", 20.0), ("rkg2", 20.0), ("backward_euler", 20.0)]


@pytest.mark.parametrize("kind,ratio", SCHEMES)
@pytest.mark.parametrize("use_ptl", [False, True])
def test_acceptance9_conservation(kind, ratio, use_ptl):
    """Criterion 9: Neumann (zero-flux) scalar diffusion conserves the
    rho V-weighted sum to 1e-12 relative over 100 outer steps."""
    x = np.linspace(0.0, 1.0, 24)
    geoms = [build_geometry([x, x], [("neumann", "neumann")] * 2),
             build_geometry([np.linspace(1.0, 2.0, 10), (np.arange(8) + 0.5) * np.pi / 8,
                             np.arange(16) * 2 * np.pi / 16],
                            [("neumann", "neumann"), ("axis", "axis"), ("periodic", "periodic")], "spherical")]
    for g in geoms:
        op = _op(g)
        W = op.weights()
        u = np.random.default_rng(9).random(g.shape)[None]
        s0 = float(np.sum(W * u))
        dt = ratio * op.euler_dt()
        for _ in range(100):
            # (BE iterates conserve only to the PCG tolerance: solve below the 1e-12 bar)
            u, _ = optl.cycle_operator(op, optl.OracleScheme(kind, tol=1e-13), u, dt, use_ptl=use_ptl)
        assert abs(float(np.sum(W * u)) - s0) <= 1e-12 * abs(s0)


@pytest.mark.parametrize("kind", ["euler", "backward_euler", "rkl2", "rkg2"])
def test_acceptance8_schemes_converge_to_fine_euler(kind):
    """Criterion 8: on a smooth 2-D anisotropic-conduction
    problem every scheme converges to the fine-Euler oracle as dt -> 0: the
    final max-norm error decreases monotonically over 3 halvings and is
    below 1e-6 at the finest dt."""
    from acceptance_cases import ANISO_STEPS, aniso_problem, aniso_reference
    dtE, ref, op = aniso_reference()
    _, u0, _ = aniso_problem()
    errs = []
    for m in ANISO_STEPS:
        u = u0.reshape((1,) + op.geom.shape)
        for _ in range(m):
            u, _ = optl.cycle_operator(op, optl.OracleScheme(kind, tol=1e-13), u, dtE / m, use_ptl=False)
        errs.append(float(np.max(np.abs(u.reshape(ref.shape) - ref))))
    assert all(b < a for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-6, errs
