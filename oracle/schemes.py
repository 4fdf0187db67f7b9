"""Oracle time integrators and PCG (test infrastructure; see oracle/__init__.py).

* RKL2 (Meyer, Balsara & Aslam 2014, the "standard published formulation"
  SPEC.md:279, :313): s = ceil((sqrt(9 + 16 dt/dtE) - 1)/2), floor 2.
* RKG2, alpha = 3/2 (Appendix A, :222-267):
  s = ceil(sqrt(25 + 24 dt/dtE)/2 - 3/2), made odd, floor 3.
* Shared s-stage recurrence:
  u_k = mu u_{k-1} + nu u_{k-2} + (1-mu-nu) u_0 + mu~ dt F(u_{k-1}) + gamma~ dt y_0,
  evaluated as ((((mu*a + nu*b) + kap*u0) + mtdt*F) + gtdt*y0) with
  kap = (1 - mu) - nu, mtdt = mu~*dt, gtdt = gamma~*dt (host doubles);
  pinned nodes copy u_0 exactly (mesh.py:5-7).
* Backward Euler + Jacobi PCG in the rho*V
  weighted inner product, x0 = u^n, convergence
  ||r||_w / ||b||_w <= tol tested after every iteration.
"""
from __future__ import annotations

import math

import numpy as np


class BlowUpError(FloatingPointError):
    def __init__(self, stage):
        super().__init__(f"non-finite value at stage {stage}")
        self.stage = stage


class IndefiniteOperatorError(ArithmeticError):
    pass


class DivergenceError(ArithmeticError):
    pass


# ---------------------------------------------------------------- counts

def rkl2_iteration_count(dt, dt_euler, make_odd=False):
    r = dt / dt_euler
    s = math.ceil((math.sqrt(9.0 + 16.0 * r) - 1.0) / 2.0)
    if make_odd and s % 2 == 0:
        s += 1
    return max(int(s), 2)


def rkg2_iteration_count(dt, dt_euler):
    r = dt / dt_euler
    s = math.ceil(0.5 * math.sqrt(25.0 + 24.0 * r) - 1.5)
    s = int(s)
    if s % 2 == 0:
        s += 1
    return max(s, 3)


# ---------------------------------------------------------------- tables

def rkl2_coefficients(s):
    """Return (mu, nu, mut, gam) lists indexed 1..s (index 0 unused)."""
    if s < 2:
        raise ValueError("RKL2 needs s >= 2")
    b = [0.0] * (s + 1)
    for j in range(s + 1):
        b[j] = 1.0 / 3.0 if j <= 2 else (j * j + j - 2.0) / (2.0 * j * (j + 1.0))
    w1 = 4.0 / (s * s + s - 2.0)
    mu = [0.0] * (s + 1)
    nu = [0.0] * (s + 1)
    mut = [0.0] * (s + 1)
    gam = [0.0] * (s + 1)
    mut[1] = b[1] * w1
    for j in range(2, s + 1):
        mu[j] = (2.0 * j - 1.0) / j * b[j] / b[j - 1]
        nu[j] = -(j - 1.0) / j * b[j] / b[j - 2]
        mut[j] = mu[j] * w1
        gam[j] = -(1.0 - b[j - 1]) * mut[j]
    return mu, nu, mut, gam


def rkg2_coefficients(s):
    """PAPER.md Appendix A with alpha = 3/2; (mu, nu, mut, gam) 1..s."""
    if s < 3 or s % 2 == 0:
        raise ValueError("RKG2 needs odd s >= 3 (SPEC.md:264)")
    w = 6.0 / ((s + 4.0) * (s - 1.0))
    b = [0.0] * (s + 1)
    b[0], b[1], b[2] = 1.0, 1.0 / 3.0, 1.0 / 15.0
    mu = [0.0] * (s + 1)
    nu = [0.0] * (s + 1)
    mut = [0.0] * (s + 1)
    gam = [0.0] * (s + 1)
    mu[1] = 1.0
    mut[1] = w
    mu[2] = 0.5
    nu[2] = -0.1
    mut[2] = mu[2] * w
    gam[2] = 0.0
    for k in range(3, s + 1):
        b[k] = 4.0 * (k - 1.0) * (k + 4.0) / (3.0 * k * (k + 1.0) * (k + 2.0) * (k + 3.0))
        mu[k] = (2.0 + 1.0 / k) * b[k] / b[k - 1]
        nu[k] = -(1.0 / k + 1.0) * b[k] / b[k - 2]
        mut[k] = mu[k] * w
        gam[k] = (k * (k + 1.0) / 2.0 * b[k - 1] - 1.0) * mut[k]
    return mu, nu, mut, gam


def stage_table(kind, s, dt):
    """Per-stage doubles (mu, nu, kap, mtdt, gtdt) for k = 1..s."""
    mu, nu, mut, gam = (rkl2_coefficients if kind == "rkl2" else rkg2_coefficients)(s)
    rows = []
    for k in range(1, s + 1):
        kap = (1.0 - mu[k]) - nu[k]
        rows.append((mu[k], nu[k], kap, mut[k] * dt, gam[k] * dt))
    return rows


# ---------------------------------------------------------------- STS step

def sts_step(apply, u0, y0, dt, s, kind, pinned):
    """s-stage recurrence; ``apply(u) -> F(u)``; ``y0 = F(u0)`` (already
    evaluated by the PTL)."""
    tab = stage_table(kind, s, dt)
    u1 = u0 + tab[0][3] * y0
    u1[..., pinned] = u0[..., pinned]
    if not np.all(np.isfinite(u1)):
        raise BlowUpError(1)
    um2, um1 = u0, u1
    for k in range(2, s + 1):
        mu, nu, kap, mtdt, gtdt = tab[k - 1]
        Fk = apply(um1)
        uk = ((((mu * um1) + (nu * um2)) + (kap * u0)) + (mtdt * Fk)) + (gtdt * y0)
        uk[..., pinned] = u0[..., pinned]
        if not np.all(np.isfinite(uk)):
            raise BlowUpError(k)
        um2, um1 = um1, uk
    return um1


def euler_step(apply, u, dt, pinned):
    out = u + dt * apply(u)
    out[..., pinned] = u[..., pinned]
    return out


# ---------------------------------------------------------------- PCG

def wdot(W, x, y):
    return float(np.sum((W * x) * y))


def pcg_solve(A, b, dinv_apply, x0, W, tol, max_iter):
    """Jacobi-PCG in the W-weighted inner product.  Returns
    (x, iterations, final_relative_residual, converged)."""
    x = x0.copy()
    r = b - A(x)
    z = dinv_apply(r)
    p = z.copy()
    rz = wdot(W, r, z)
    bn = math.sqrt(wdot(W, b, b))
    rel = float("inf")
    it = 0
    converged = False
    for it in range(1, max_iter + 1):
        Ap = A(p)
        pAp = wdot(W, p, Ap)
        if rz != 0.0:
            if not pAp > 0.0:
                if math.isnan(pAp):
                    raise DivergenceError("NaN in PCG")
                raise IndefiniteOperatorError("p^T A p <= 0 in PCG")
            alpha = rz / pAp
        else:
            alpha = 0.0
        x = x + alpha * p
        r = r - alpha * Ap
        rr = wdot(W, r, r)
        if not math.isfinite(rr):
            raise DivergenceError("non-finite residual in PCG")
        rn = math.sqrt(rr)
        rel = rn / bn if bn > 0.0 else (0.0 if rn == 0.0 else float("inf"))
        if rel <= tol:
            converged = True
            break
        z = dinv_apply(r)
        rz_new = wdot(W, r, z)
        beta = rz_new / rz if rz != 0.0 else 0.0
        p = z + beta * p
        rz = rz_new
    return x, it, rel, converged


def backward_euler_step(apply, diag, W, u, dt, tol, max_iter, pinned, line=None):
    """Solve (I - dt J) x = u with x0 = u; ``diag`` = -J_ii (pinned rows 0).
    ``line`` = (jl, ju): the r-line preconditioner (-J_{i,i-1}, -J_{i,i+1},
    single component) instead of point Jacobi."""
    dvec = 1.0 + dt * diag
    inv = 1.0 / dvec  # the stored inverse diagonal, once per solve

    def A(x):
        return x - dt * apply(x)

    if line is None:
        def dinv(r):
            return r * inv
    else:
        from .operators import line_factor, line_solve
        jl, ju = line
        inv, cp = line_factor(1.0, diag[0], jl, ju, dt)

        def dinv(r):
            return line_solve(r[0], jl, inv, cp, dt)[None]

    return pcg_solve(A, u, dinv, u, W, tol, max_iter)
