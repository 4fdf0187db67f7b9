"""Von Neumann amplification, STS speed-up, convergence studies and the
fine-Euler reference (the machinery behind PAPER.md Fig. 1).

Convention (SPEC.md:479 open question, fixed here): theta = k dx in (0, pi],
1-D uniform second-order central difference, lambda(theta) = (4/dx^2)
sin^2(theta/2), dt = r dt_E with dt_E = dx^2/2, so z = dt lambda = 2 r
sin^2(theta/2) (= 2r at theta = pi, the SPEC's closed-form check).

Two evaluations of every amplification factor, as the SPEC asks
(SPEC.md:461, :467-468):

* ``amplification`` -- closed form: BE 1/(1+z), exact e^{-z}, STS by running
  the stage recurrence on the scalar mode u' = -(z/dt) u with the production
  coefficient tables (pc_sts_table);
* ``amplification_run`` -- the production GPU path itself: one step of the
  scheme on a 1-D periodic grid of 2*M nodes (``schemes.step_*``) applied to
  a field with every Fourier mode present; the amplification of mode m is
  the ratio of its discrete Fourier coefficients after / before (the modes
  are exact eigenvectors of the periodic 3-point operator), theta_m = pi m/M.
"""
from __future__ import annotations

import math

import numpy as np

from . import mesh, operators, schemes

SCHEMES = ("be", "rkl2", "rkg2", "exact", "euler")


def _z(r, theta):
    return 2.0 * r * np.sin(np.asarray(theta, float) / 2.0) ** 2


def stage_count(kind, r):
    if kind == "rkg2":
        return schemes.rkg2_iteration_count(float(r), 1.0)
    return schemes.rkl2_iteration_count(float(r), 1.0)


def _sts_scalar(kind, z, s):
    """The s-stage recurrence on u' = -lam u with dt lam = z (elementwise in z)."""
    tab = schemes.sts_table(kind, s, 1.0)  # (mu, nu, kap, mt dt, gt dt) with dt = 1
    z = np.asarray(z, float)
    u0 = np.ones_like(z)
    y0 = -z * u0
    um2, um1 = u0, u0 + tab[0, 3] * y0
    for k in range(2, s + 1):
        mu, nu, kap, mt, gt = tab[k - 1]
        um2, um1 = um1, ((((mu * um1) + (nu * um2)) + (kap * u0)) + (mt * (-z * um1))) + (gt * y0)
    return um1


def amplification(kind, r, theta):
    """|R(z(theta))| for scheme ``kind`` at dt = r dt_E (closed form / scalar recurrence)."""
    if kind not in SCHEMES:
        raise ValueError(f"unknown scheme {kind!r}")
    if not r > 0:
        raise ValueError("r must be > 0")
    z = _z(r, theta)
    if kind == "be":
        return np.abs(1.0 / (1.0 + z))
    if kind == "exact":
        return np.exp(-z)
    if kind == "euler":
        return np.abs(1.0 - z)
    return np.abs(_sts_scalar(kind, z, stage_count(kind, r)))


def exact_amplification(r, theta):
    return amplification("exact", r, theta)


def _periodic_problem(M):
    n = 2 * M
    g = mesh.build_grid([n], coords=[np.arange(n, dtype=float)])  # dx = 1
    bc = mesh.BoundaryCondition.periodic(1)
    op = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=bc), 1)
    return g, op


def amplification_run(kind, r, M=512, seed=0):
    """(theta_m, |R_m|) for m = 1..M from ONE device step of scheme ``kind``."""
    if kind not in ("be", "rkl2", "rkg2", "euler"):
        raise ValueError(f"scheme {kind!r} has no device step")
    g, op = _periodic_problem(M)
    n = 2 * M
    rng = np.random.default_rng(seed)
    amp = rng.uniform(0.5, 1.5, M + 1)
    ph = rng.uniform(0.0, 2.0 * math.pi, M + 1)
    i = np.arange(n)
    u0 = np.sum([amp[m] * np.cos(math.pi * m * i / M + ph[m]) for m in range(1, M + 1)], axis=0)
    dtE = 0.5
    dt = r * dtE
    f = mesh.Field(g, u0[:, None])
    if kind == "be":
        out, _ = schemes.step_backward_euler(op, f, dt, schemes.SchemeConfig("backward_euler", tol=1e-14,
                                                                              max_iter=100000))
    elif kind == "euler":
        out = schemes.step_euler(op, f, dt)
    else:
        out = (schemes.step_rkl2 if kind == "rkl2" else schemes.step_rkg2)(op, f, dt, dtE)
    a0 = np.fft.rfft(u0)[1:M + 1]
    a1 = np.fft.rfft(out.values[:, 0])[1:M + 1]
    theta = math.pi * np.arange(1, M + 1) / M
    return theta, np.abs(a1 / a0)


def speedup_estimate(kind, r):
    """r / s(r): one STS stage costed as one Euler step (Fig. 1 left)."""
    if kind not in ("rkl2", "rkg2"):
        raise ValueError("speedup is defined for rkl2 / rkg2")
    if not r >= 1.0:
        raise ValueError("r must be >= 1")
    return float(r) / stage_count(kind, r)


def convergence_study(kind, dts=None, M=32, T=None):
    """Least-squares slope of log(error) vs log(dt) for one step of ``kind`` on
    the 1-D periodic heat equation with a single sinusoidal mode (analytic
    decay e^{-lam t}); returns (order, dts, errors)."""
    g, op = _periodic_problem(M)
    n = 2 * M
    m = 3
    theta = math.pi * m / M
    lam = 4.0 * math.sin(theta / 2.0) ** 2
    i = np.arange(n)
    u0 = np.sin(theta * i)
    T = T if T is not None else 2.0
    dts = dts if dts is not None else [T / 2 ** k for k in range(3, 8)]
    errs = []
    for dt in dts:
        u = mesh.Field(g, u0[:, None].copy())
        for _ in range(int(round(T / dt))):
            if kind == "be":
                u, _ = schemes.step_backward_euler(op, u, dt, schemes.SchemeConfig("backward_euler", tol=1e-14,
                                                                                    max_iter=100000))
            elif kind == "euler":
                u = schemes.step_euler(op, u, dt)
            else:
                u = (schemes.step_rkl2 if kind == "rkl2" else schemes.step_rkg2)(op, u, dt, 0.5)
        errs.append(float(np.max(np.abs(u.values[:, 0] - math.exp(-lam * T) * u0))))
    slope = np.polyfit(np.log(dts), np.log(errs), 1)[0]
    return float(slope), list(dts), errs


def oracle_fine_euler(op, u, total_dt, n_sub):
    """n_sub explicit-Euler substeps of total_dt / n_sub (the reference-solution generator)."""
    dtE = operators.estimate_euler_dt(op, u)
    h = total_dt / n_sub
    if h > dtE:
        raise ValueError("substep exceeds the explicit stability limit")
    for _ in range(n_sub):
        u = schemes.step_euler(op, u, h)
    return u


def write_ampfactor_csv(path, kinds, r, M=512):
    theta = math.pi * np.arange(1, M + 1) / M
    with open(path, "w") as fh:
        fh.write("scheme,r,theta,amplification\n")
        for k in kinds:
            a = amplification(k, r, theta)
            for t, v in zip(theta, a):
                fh.write(f"{k},{r!r},{float(t)!r},{float(v)!r}\n")


def write_speedup_csv(path, rmin, rmax, n=50):
    if not (rmin >= 1.0 and rmax >= rmin):
        raise ValueError("need 1 <= rmin <= rmax")
    rs = np.unique(np.geomspace(rmin, rmax, n)) if rmax > rmin else np.array([rmin])
    with open(path, "w") as fh:
        fh.write("scheme,r,s,speedup\n")
        for k in ("rkl2", "rkg2"):
            for r in rs:
                fh.write(f"{k},{float(r)!r},{stage_count(k, r)},{speedup_estimate(k, r)!r}\n")
