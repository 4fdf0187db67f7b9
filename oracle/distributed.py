"""Slab-decomposed restatement of the cycle (test infrastructure; see
oracle/__init__.py) -- the algorithm the r-slab CUDA path implements
(paper_2403_01004_b200/csrc/capi_objects.cuh: halo_exchange, global_argmax;
capi_sts.cuh: ptl_device; capi_pcg.cuh: pcg_split_fin), written over ``torch.distributed`` so it runs on
CPU ranks with the gloo backend.

Per rank: the axis-0 slab [i0, i0 + n) of geometry.slab_bounds, stored with
one ghost plane on each side that has a neighbour slab.  Every operator
application exchanges the ghost planes first (send/recv of one plane per
neighbour), then evaluates the oracle operator on the extended slab with the
global metric tables sliced to it; the interior planes are bitwise those of the
single-domain evaluation because every stencil has radius 1.

PTL: local |F| argmax (lowest AoS index) -> all_gather of
(value, global index) -> the same combine on every rank -> the owner of k
evaluates the pairs with its ghost planes of u and F -> all_reduce(min).
PCG inner products are GPU-count invariant (the CUDA path's
kernels.cuh PlaneRed): every rank sums each of its axis-0 planes, the
per-plane sums are all-gathered into the global plane vector, and every rank
adds the planes in global order 0 .. n0-1 -- the same numbers in the same
order for any number of slabs, so iteration counts and fields are bitwise
identical for 1, 2, 3, 8 ... ranks.
"""
from __future__ import annotations

import copy
import math

import numpy as np
import torch
import torch.distributed as dist

from . import operators as ops
from . import schemes as sch
from .ptl import CycleRecord, _aos_argmax, step_count


def slab_bounds(n0, nranks, rank):
    """Balanced slabs: the first n0 % nranks ranks get one extra plane
    (mirrors paper_2403_01004_b200.geometry.slab_bounds)."""
    base, extra = divmod(n0, nranks)
    return rank * base + min(rank, extra), base + (1 if rank < extra else 0)


class Slab:
    def __init__(self, geom, rank, nranks):
        n0 = geom.shape[0]
        self.rank, self.nranks = rank, nranks
        self.i0, self.n = slab_bounds(n0, nranks, rank)
        per0 = geom.periodic[0]
        self.lo = rank > 0 or (per0 and nranks > 1)   # a lower neighbour slab exists
        self.hi = rank < nranks - 1 or (per0 and nranks > 1)
        self.glo, self.ghi = int(self.lo), int(self.hi)
        self.global_geom = geom
        self.geom = self._slice_geometry(geom)

    # extended-slab geometry: 2-D tables sliced with ghost rows, axis 0 not
    # periodic inside the slab (its neighbours come from the ghost planes)
    def _slice_geometry(self, g):
        n0 = g.shape[0]
        rows = [(self.i0 - self.glo + q) % n0 for q in range(self.n + self.glo + self.ghi)]
        s = copy.copy(g)
        s.shape = (len(rows),) + tuple(g.shape[1:])
        s.periodic = (False,) + tuple(g.periodic[1:])
        take = lambda t: np.ascontiguousarray(np.asarray(t)[rows])  # noqa: E731
        s.W2 = [take(t) for t in g.W2]
        s.iV2, s.V2 = take(g.iV2), take(g.V2)
        s.iL2 = {k: take(v) for k, v in g.iL2.items()}
        s.wo01 = {k: take(v) for k, v in g.wo01.items()}
        s.iVal2, s.Val2 = take(g.iVal2), take(g.Val2)
        pin = g.pinned[rows]
        s.__class__ = type("SlabGeometry", (g.__class__,), {"pinned": property(lambda self_: pin)})
        return s

    def interior(self, a):
        return a[..., self.glo:self.glo + self.n, :, :]

    def extend(self, interior_values):
        """(ncomp, n, n1, n2) -> (ncomp, n + ghosts, n1, n2), ghosts zero."""
        c, n, n1, n2 = interior_values.shape
        out = np.zeros((c, n + self.glo + self.ghi, n1, n2))
        out[:, self.glo:self.glo + n] = interior_values
        return out

    def halo(self, ext):
        """Exchange the ghost planes of an extended (ncomp, n+g, n1, n2) array."""
        P, r = self.nranks, self.rank
        if P == 1:
            return ext
        reqs = []
        lo_rank, hi_rank = (r - 1) % P, (r + 1) % P
        recv_lo = torch.empty(ext.shape[0], *ext.shape[2:], dtype=torch.float64) if self.lo else None
        recv_hi = torch.empty(ext.shape[0], *ext.shape[2:], dtype=torch.float64) if self.hi else None
        first = torch.from_numpy(np.ascontiguousarray(ext[:, self.glo]))
        last = torch.from_numpy(np.ascontiguousarray(ext[:, self.glo + self.n - 1]))
        if self.lo:
            reqs.append(dist.isend(first, lo_rank))
            reqs.append(dist.irecv(recv_lo, lo_rank))
        if self.hi:
            reqs.append(dist.isend(last, hi_rank))
            reqs.append(dist.irecv(recv_hi, hi_rank))
        for q in reqs:
            q.wait()
        if self.lo:
            ext[:, 0] = recv_lo.numpy()
        if self.hi:
            ext[:, -1] = recv_hi.numpy()
        return ext

    def plane_sum(self, prod):
        """Sum of an (ncomp, n, n1, n2) interior array in the slab-invariant
        order: per plane, then over the GLOBAL planes in index order."""
        local = [float(np.sum(prod[:, q])) for q in range(prod.shape[1])]
        n0 = self.global_geom.shape[0]
        if self.nranks > 1:
            vec = torch.zeros(n0, dtype=torch.float64)
            vec[self.i0:self.i0 + self.n] = torch.tensor(local, dtype=torch.float64)
            dist.all_reduce(vec)  # one non-zero contribution per entry: exact
            planes = vec.tolist()
        else:
            planes = local
        s = 0.0
        for v in planes:
            s += v
        return s

    def all_sum(self, x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    def all_min(self, x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return float(t.item())

    def all_max(self, x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())


class SlabOperator:
    """Wraps an oracle operator (built on the GLOBAL geometry) for a slab."""

    def __init__(self, op, slab):
        self.slab = slab
        self.op = copy.copy(op)
        self.op.geom = slab.geom
        rows = slice(None)
        n0 = op.geom.shape[0]
        idx = [(slab.i0 - slab.glo + q) % n0 for q in range(slab.n + slab.glo + slab.ghi)]
        for name in ("D", "rho", "c"):
            v = getattr(op, name)
            if isinstance(v, np.ndarray) and v.ndim == 3:
                setattr(self.op, name, np.ascontiguousarray(v[idx]))
        if op.b is not None:
            self.op.b = np.ascontiguousarray(op.b[:, idx])
        del rows

    def apply_ext(self, u_ext):
        """F on the interior planes, from an extended array (ghosts exchanged here)."""
        self.slab.halo(u_ext)
        return self.slab.interior(self.op.apply(u_ext))

    def euler_dt(self):
        lam, _ = self.op.bound_and_diag()
        m = float(np.max(self.slab.interior(lam))) if lam.size else 0.0
        m = self.slab.all_max(m)
        return float("inf") if not m > 0.0 else 2.0 / m


def slab_compute_ptl(sop, u_ext, F_int, eps_rel=1e-12):
    slab, g = sop.slab, sop.slab.global_geom
    ncomp = F_int.shape[0]
    c_k, k_loc, flat = _aos_argmax(np.abs(F_int))
    v = float(np.abs(F_int)[(c_k,) + k_loc])
    gidx = flat + slab.i0 * g.shape[1] * g.shape[2] * ncomp  # global AoS index
    pairs = [torch.zeros(2, dtype=torch.float64) for _ in range(slab.nranks)]
    dist.all_gather(pairs, torch.tensor([v, float(gidx)], dtype=torch.float64))
    best_v, best_i = -1.0, None
    for p in pairs:
        pv, pi = float(p[0]), int(p[1])
        if pv > best_v or (pv == best_v and pi < best_i):
            best_v, best_i = pv, pi
    thr = eps_rel * best_v
    pt = best_i // ncomp
    kk = pt % g.shape[2]
    kj = (pt // g.shape[2]) % g.shape[1]
    ki = pt // (g.shape[2] * g.shape[1]) - slab.i0
    best = math.inf
    F_ext = slab.halo(slab.extend(F_int))  # every rank exchanges F's ghost planes
    if 0 <= ki < slab.n:  # owner of k
        e = ki + slab.glo
        for a in range(3):
            n = g.shape[a]
            if n == 1:
                continue
            for d in (-1, 1):
                q = [e, kj, kk]
                q[a] += d
                if a == 0:
                    if q[0] < 0 or q[0] >= F_ext.shape[1]:
                        continue
                    if (q[0] < slab.glo and not slab.lo) or (q[0] >= slab.glo + slab.n and not slab.hi):
                        continue
                else:
                    if q[a] < 0 or q[a] >= n:
                        if not g.periodic[a]:
                            continue
                        q[a] %= n
                for c in range(ncomp):
                    du = float(u_ext[(c, e, kj, kk)]) - float(u_ext[(c,) + tuple(q)])
                    dF = float(F_ext[(c, e, kj, kk)]) - float(F_ext[(c,) + tuple(q)])
                    if du != 0.0 and abs(dF) > thr and du * dF < 0.0:
                        best = min(best, -du / dF)
    best = slab.all_min(best)
    return None if math.isinf(best) else best


def slab_cycle_operator(sop, kind, u_int, outer_dt, dt_euler, eps_rel=1e-12, tol=1e-10, max_iter=10000,
                        max_cycles=None):
    """oracle.ptl.cycle_operator over slabs (RKL2/RKG2 or BE+PCG);
    ``max_cycles``: stop after that many cycles (partial step)."""
    slab = sop.slab
    pinned = slab.interior(slab.geom.pinned[None])[0]
    report = []
    remaining = float(outer_dt)
    u = u_int.copy()
    cyc = 0
    scheme = type("S", (), {"kind": kind, "make_odd": False})()
    while remaining > 0.0 and (max_cycles is None or cyc < max_cycles):
        u_ext = slab.extend(u)
        F = sop.apply_ext(u_ext)
        ptl = slab_compute_ptl(sop, u_ext, F, eps_rel)
        if ptl is None:
            dt = remaining
        else:
            dt = max(ptl, dt_euler)
            if dt >= remaining:
                dt = remaining
        if kind in ("rkl2", "rkg2"):
            s = step_count(scheme, dt, dt_euler)
            u = sch.sts_step(lambda x: sop.apply_ext(slab.extend(x)), u, F, dt, s, kind, pinned)
            iters = s
        else:
            _, diag = sop.op.bound_and_diag()
            dvec = 1.0 + dt * slab.interior(diag)
            W = slab.interior(sop.op.weights())
            wdot = lambda x, y: slab.plane_sum((W * x) * y)  # noqa: E731
            A = lambda x: x - dt * sop.apply_ext(slab.extend(x))  # noqa: E731
            inv = 1.0 / dvec  # the stored inverse diagonal
            u, iters = _pcg(A, u, lambda r: r * inv, u, wdot, tol, max_iter)
        cyc += 1
        report.append(CycleRecord(cyc, dt, ptl, ptl is not None, iters))
        remaining = 0.0 if dt == remaining else remaining - dt
    return u, report


def _pcg(A, b, dinv, x0, wdot, tol, max_iter):
    x = x0.copy()
    r = b - A(x)
    z = dinv(r)
    p = z.copy()
    rz = wdot(r, z)
    bn = math.sqrt(wdot(b, b))
    it = 0
    for it in range(1, max_iter + 1):
        Ap = A(p)
        pAp = wdot(p, Ap)
        alpha = rz / pAp if rz != 0.0 else 0.0
        x = x + alpha * p
        r = r - alpha * Ap
        rn = math.sqrt(wdot(r, r))
        if (rn / bn if bn > 0 else 0.0) <= tol:
            break
        z = dinv(r)
        rz_new = wdot(r, z)
        beta = rz_new / rz if rz != 0.0 else 0.0
        p = z + beta * p
        rz = rz_new
    return x, it
