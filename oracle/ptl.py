"""Oracle PTL, cycling controller and split driver (test infrastructure).

* ``compute_ptl``    -- PAPER.md Eq. 3-5 (:57-74), SPEC.md:345-353, :380-384:
  k = argmax |F| over points x components, ties -> lowest linear index of the
  reference Field layout (point-major, component innermost); for every
  existing orthogonal neighbour and every component, with du = u_k - u_nb and
  dF = F_k - F_nb: if du != 0, |dF| > eps_rel*max|F| and du*dF < 0, candidate
  -du/dF; the minimum, or None ("unlimited").  ``check_all`` scans all pairs.
  Neighbours across non-periodic faces and across the pole do not exist.
* ``cycle_operator`` -- SPEC.md:354-362, :381: dt_c = min(max(ptl, floor),
  remaining), unlimited -> all remaining; y0 of the STS step is the F the PTL
  just used; the last cycle takes exactly the remainder.
* ``split_advance``  -- SPEC.md:363-371, :385-386: Lie splitting in list order,
  lagged T0 refreshed once per outer step.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import operators as ops
from . import schemes as sch


class CycleCapError(RuntimeError):
    def __init__(self, report):
        super().__init__(f"max_cycles reached after {len(report)} cycles")
        self.report = report


@dataclass
class OracleOperator:
    """Frozen linear operator over SoA fields (ncomp, n0, n1, n2)."""

    geom: object
    kind: str  # "scalar" | "aligned"
    ncomp: int = 1
    D: object = None
    rho: object = None
    vector_metric: bool = False
    b: object = None
    c: object = None
    pref: float = 1.0

    def apply(self, u):
        if self.kind == "scalar":
            return ops.scalar_apply(self.geom, u, self.D, self.rho, self.vector_metric)
        return ops.aligned_apply(self.geom, u[0], self.b, self.c, self.rho, self.pref)[None]

    def bound_and_diag(self):
        if self.kind == "scalar":
            lam = ops.scalar_gershgorin(self.geom, self.D, self.rho, self.ncomp, self.vector_metric)
            dg = ops.scalar_diag(self.geom, self.D, self.rho)
            return lam, np.broadcast_to(dg, (self.ncomp,) + dg.shape)
        lam, dg = ops.aligned_gershgorin(self.geom, self.b, self.c, self.rho, self.pref)
        return lam[None], dg[None]

    def euler_dt(self):
        lam, _ = self.bound_and_diag()
        return ops.euler_dt(lam)

    def line_offdiag(self):
        """(-J_{i,i-1}, -J_{i,i+1}) for the r-line preconditioner (aligned only)."""
        if self.kind != "aligned":
            raise NotImplementedError("the r-line preconditioner is built for the aligned operator")
        return ops.aligned_line_offdiag(self.geom, self.b, self.c, self.rho, self.pref)

    def weights(self):
        V = self.geom.volume() if self.kind == "scalar" else self.geom.aligned_volume()
        W = V if self.rho is None else self.rho * V
        return np.broadcast_to(W, (self.ncomp,) + W.shape)


def _aos_argmax(absF):
    """Lowest AoS linear index of the maximum (numpy argmax = first hit)."""
    aos = np.moveaxis(absF, 0, -1)
    flat = int(np.argmax(aos))
    ncomp = absF.shape[0]
    c = flat % ncomp
    pt = np.unravel_index(flat // ncomp, absF.shape[1:])
    return c, pt, flat


def neighbours(geom, pt):
    out = []
    for a in range(3):
        n = geom.shape[a]
        if n == 1:
            continue
        for d in (-1, 1):
            q = list(pt)
            q[a] += d
            if q[a] < 0 or q[a] >= n:
                if not geom.periodic[a]:
                    continue
                q[a] %= n
            out.append(tuple(q))
    return out


def compute_ptl(u, F, geom, eps_rel=1e-12, check_all=False):
    absF = np.abs(F)
    c_k, k, flat = _aos_argmax(absF)
    fmax = float(absF[(c_k,) + k])
    thr = eps_rel * fmax
    if check_all:
        return _ptl_all(u, F, geom, thr)
    best = None
    for nb in neighbours(geom, k):
        for c in range(u.shape[0]):
            du = float(u[(c,) + k]) - float(u[(c,) + nb])
            dF = float(F[(c,) + k]) - float(F[(c,) + nb])
            if du != 0.0 and abs(dF) > thr and du * dF < 0.0:
                cand = -du / dF
                if best is None or cand < best:
                    best = cand
    return best


def _ptl_all(u, F, geom, thr):
    best = None
    for a in range(3):
        n = geom.shape[a]
        if n == 1:
            continue
        up = ops.shift(u, a, 1, geom.periodic[a])
        Fp = ops.shift(F, a, 1, geom.periodic[a])
        du = u - up
        dF = F - Fp
        ok = (du != 0.0) & (np.abs(dF) > thr) & (du * dF < 0.0)
        if np.any(ok):
            m = float(np.min(-du[ok] / dF[ok]))
            best = m if best is None else min(best, m)
    return best


@dataclass
class CycleRecord:
    cycle: int
    dt: float
    ptl_raw: object  # float or None (unlimited)
    limited: bool
    iters: int  # s (STS) or PCG iterations


@dataclass
class OracleScheme:
    kind: str  # rkl2 | rkg2 | backward_euler | euler
    tol: float = 1e-10
    max_iter: int = 10000
    make_odd: bool = False
    preconditioner: str = "jacobi"  # or "line-r" (aligned / scalar one-component operators)


def step_count(scheme, dt, dt_euler):
    if scheme.kind == "rkl2":
        return sch.rkl2_iteration_count(dt, dt_euler, scheme.make_odd)
    return sch.rkg2_iteration_count(dt, dt_euler)


def cycle_operator(op, scheme, u, outer_dt, eps_rel=1e-12, floor="euler", floor_fraction=1.0,
                   max_cycles=10**6, check_all=False, use_ptl=True, dt_euler=None, static=False,
                   refresh_cycle=None):
    """``use_ptl`` False: one cycle of the whole step.  ``static``: first-PTL
    cycling -- the first cycle's PTL is reused by every later cycle
    (SPEC.md:362).  ``refresh_cycle(op, u)``: re-freeze the lagged T0 := u at
    the start of every cycle (SPEC.md:385 per-cycle knob); Delta t_E (unless
    given) and the BE diagonal follow the refreshed operator."""
    fixed_dtE = dt_euler is not None
    if dt_euler is None:
        dt_euler = op.euler_dt()
    pinned = op.geom.pinned
    floor_dt = dt_euler if floor == "euler" else floor_fraction * dt_euler
    report = []
    remaining = float(outer_dt)
    diag = W = None
    if scheme.kind == "backward_euler":
        _, diag = op.bound_and_diag()
        W = op.weights()
    cyc = 0
    first_ptl = None
    while remaining > 0.0:
        if cyc >= max_cycles:
            raise CycleCapError(report)
        if refresh_cycle is not None:
            refresh_cycle(op, u)
            if not fixed_dtE:
                dt_euler = op.euler_dt()
                floor_dt = dt_euler if floor == "euler" else floor_fraction * dt_euler
            if scheme.kind == "backward_euler":
                _, diag = op.bound_and_diag()
        F = op.apply(u)
        if use_ptl and (not static or cyc == 0):
            ptl = compute_ptl(u, F, op.geom, eps_rel, check_all)
            first_ptl = ptl
        else:
            ptl = first_ptl if use_ptl else None
        if ptl is None:
            dt = remaining
        else:
            dt = max(ptl, floor_dt)
            if dt >= remaining:
                dt = remaining
        if scheme.kind in ("rkl2", "rkg2"):
            s = step_count(scheme, dt, dt_euler)
            u = sch.sts_step(op.apply, u, F, dt, s, scheme.kind, pinned)
            iters = s
        elif scheme.kind == "backward_euler":
            line = op.line_offdiag() if scheme.preconditioner == "line-r" else None
            u, iters, rel, conv = sch.backward_euler_step(
                op.apply, diag, W, u, dt, scheme.tol, scheme.max_iter, pinned, line=line)
        else:
            un = u + dt * F
            un[..., pinned] = u[..., pinned]  # pinned (Dirichlet) nodes keep u0 exactly
            u = un
            iters = 1
        cyc += 1
        report.append(CycleRecord(cyc, dt, ptl, ptl is not None, iters))
        if dt == remaining:
            remaining = 0.0
        else:
            remaining = remaining - dt
    return u, report


def split_advance(ops, state, outer_dt, schemes, refresh=None, eps_rel=1e-12):
    """Lie splitting in list order: ``ops`` = [(name,
    OracleOperator)], ``state`` = {name: SoA array}.  Aligned operators get
    c = aligned_coefficient(T0) from the state at the START of the outer step
    (lagged T0) through ``refresh(op, state)``.  Returns (state,
    [report per operator])."""
    state = dict(state)
    for name, op in ops:
        if op.kind == "aligned" and refresh is not None:
            refresh(op, state)
    reports = []
    for (name, op), scheme in zip(ops, schemes):
        state[name], rep = cycle_operator(op, scheme, state[name], outer_dt, eps_rel=eps_rel)
        reports.append(rep)
    return state, reports
