"""Problems of the SPEC's acceptance criteria 4-6 and 9,
shared by the oracle tests (test_oracle_acceptance.py) and the GPU tests
(test_gpu_acceptance.py)."""
from __future__ import annotations

import numpy as np

from oracle.geometry import build_geometry

# the two step problems of criteria 4 and 6 (1-D and 2-D, Neumann faces)
STEP_CASES = [(1, 64), (2, 32)]
RATIO = 500.0  # outer_dt = 500 dt_E


def coords(dim, n):
    return [np.linspace(0.0, 1.0, n)] * dim


def step_values(dim, n):
    """Step initial data: 1 on the lower half (1-D) / lower-left quadrant (2-D)."""
    u = np.zeros((n,) * dim)
    u[(slice(0, n // 2),) * dim] = 1.0
    return u


def oracle_geom(dim, n, kind="neumann"):
    return build_geometry(coords(dim, n), [(kind, kind)] * dim)


def sign_changes(u):
    """Number of adjacent-difference sign changes along every axis (the
    oscillation count of SPEC.md:550; zero differences do not count)."""
    u = np.asarray(u, float)
    total = 0
    for a in range(u.ndim):
        d = np.diff(u, axis=a)
        m = d.shape[a]
        d1 = np.take(d, range(m - 1), axis=a)
        d2 = np.take(d, range(1, m), axis=a)
        total += int(np.sum(d1 * d2 < 0.0))
    return total


def random_fields(count, seed=5):
    """Seeded random fields of criterion 5: alternately 1-D (n = 32) and
    2-D (12 x 12), Gaussian values, some with a smooth background."""
    rng = np.random.default_rng(seed)
    for q in range(count):
        if q % 2 == 0:
            n = (32,)
        else:
            n = (12, 12)
        u = rng.normal(size=n)
        if q % 4 == 3:
            u = u * 0.1 + np.linspace(0.0, 3.0, n[0]).reshape((-1,) + (1,) * (len(n) - 1))
        yield u


def neighbours(shape, k):
    out = []
    for a in range(len(shape)):
        for d in (-1, 1):
            q = list(k)
            q[a] += d
            if 0 <= q[a] < shape[a]:
                out.append(tuple(q))
    return out


# ---- criterion 8: smooth 2-D anisotropic conduction (b at 30 degrees to x,
# periodic unit square, c = 1), one outer time T = dt_E, every scheme at
# T/16 .. T/128 against a fine explicit Euler (T / 2^16)
ANISO_N = 24
ANISO_STEPS = (16, 32, 64, 128)
ANISO_FINE = 1 << 16


def aniso_problem():
    import math
    x = np.arange(ANISO_N) / ANISO_N
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = 0.1 * np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y) + 0.05 * np.cos(2 * np.pi * (X + Y))
    b = np.zeros((ANISO_N, ANISO_N, 3))
    b[..., 0] = math.cos(math.pi / 6)
    b[..., 1] = math.sin(math.pi / 6)
    return x, u0, b


_FINE = {}


def aniso_reference():
    """Fine explicit Euler (oracle) of the criterion-8 problem: (dt_E, u(T))."""
    if "ref" not in _FINE:
        from oracle import operators as oops
        from oracle import ptl as optl
        from oracle import schemes as osch
        x, u0, b = aniso_problem()
        g = build_geometry([x, x], [("periodic", "periodic")] * 2)
        op = optl.OracleOperator(g, "aligned", 1, None, None, False, np.moveaxis(b, -1, 0)[..., None],
                                 oops.aligned_coefficient(np.ones(g.shape)), 1.0)
        dtE = op.euler_dt()
        u = u0.reshape((1,) + g.shape)
        for _ in range(ANISO_FINE):
            u = osch.euler_step(op.apply, u, dtE / ANISO_FINE, g.pinned)
        _FINE["ref"] = (dtE, u.reshape(u0.shape), op)
    return _FINE["ref"]
