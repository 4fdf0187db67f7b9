"""Metric tables of the discretisation, packed for the C ABI.

Host-side numpy, computed once per (grid, boundary condition) and uploaded,
so the device and any checker see identical bits.  The
mathematics:

  scalar 7-point FV   face (+) coefficient = W2[a][i, j] * g1[a][k],
                      control volume       = V2[i, j] * gv[k]
  aligned 19-point    one-sided inverse edge lengths iL2[(a,s)][i,j] * iL1[(a,s)][k],
                      corner-tetrahedron octant weights wo01[(s0,s1)][i,j] * wo2[s2][k]
  vector metric       per-theta-row frame rotations M[face] (3x3) and the
                      Gershgorin row factors Rabs = 1 + sum_b |M[a][b]|

Cartesian tables reproduce the reference dual cells (mesh.py:130-156):
volume == Grid.dual_volumes(bc).

TABLE_ORDER (the layout pc_grid_create expects; A = (n0 + 2) x n1 with
axis-0 ghost rows, K = n2, J = n1):
  W2[0..2] (A)  g1[0..2] (K)  iV2 (A)  igv (K)
  iL2[(a,s)] a=0..2, s=+,- (6 A)   iL1[(a,s)] (6 K)
  wo01[++,+-,-+,--] (4 A)  wo2[+,-] (2 K)  iVal2 (A)  iValg (K)
  M[t+,t-,p+,p-] (4 x J x 9)  Rabs[t+,t-,p+,p-] (4 x J x 3)
  V2 (A)  gv (K)  Val2 (A)  Valg (K)
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import mesh

FACES = ("t+", "t-", "p+", "p-")
SIGNS = ("+", "-")
NFLAGS = 17


def _isin(kind):
    return kind


def _sin(x):
    return np.array([math.sin(v) for v in np.ravel(x)]).reshape(np.shape(x))


def _cos(x):
    return np.array([math.cos(v) for v in np.ravel(x)]).reshape(np.shape(x))


def _inv_where(h, ok):
    out = np.zeros_like(h)
    out[ok] = 1.0 / h[ok]
    return out


def _axis_info(x, periodic):
    """(+ spacing, - spacing, has +, has -) per node; periodic seam uses the
    mean edge spacing (reference mesh.py:130-133)."""
    n = x.size
    hp = np.zeros(n)
    hm = np.zeros(n)
    okp = np.zeros(n, bool)
    okm = np.zeros(n, bool)
    if n > 1:
        d = x[1:] - x[:-1]
        hp[:-1] = d
        hm[1:] = d
        okp[:-1] = True
        okm[1:] = True
        if periodic:
            seam = 0.5 * (d[0] + d[-1])
            hp[-1] = seam
            hm[0] = seam
            okp[-1] = True
            okm[0] = True
    return hp, hm, okp, okm


def _dual(x, periodic):
    n = x.size
    if n == 1:
        return np.ones(1)
    d = x[1:] - x[:-1]
    w = np.empty(n)
    w[1:-1] = 0.5 * (d[:-1] + d[1:])
    if periodic:
        seam = 0.5 * (d[0] + d[-1])
        w[0] = 0.5 * (seam + d[0])
        w[-1] = 0.5 * (d[-1] + seam)
    else:
        w[0] = 0.5 * d[0]
        w[-1] = 0.5 * d[-1]
    return w


@dataclass
class GlobalTables:
    shape: tuple
    spherical: bool
    periodic: tuple
    pinned: tuple  # ((lo, hi),) * 3
    two: dict      # name -> (n0, n1) array
    one: dict      # name -> (n2,) array
    rot: dict      # name -> (n1, 9) or (n1, 3)


def _kinds(grid, bc):
    """Face kinds embedded in three axes (singleton padding axes: 'none')."""
    coords = [np.asarray(c, float) for c in grid.coords]
    faces = [tuple(f) for f in bc.faces]
    if len(faces) != len(coords):
        raise ValueError("boundary condition dimensionality mismatch")
    kinds = [(lo.kind, hi.kind) for lo, hi in faces]
    while len(coords) < 3:
        coords.append(np.zeros(1))
        kinds.append(("none", "none"))
    return coords, kinds


def global_tables(grid, bc) -> GlobalTables:
    metric = getattr(grid, "metric", mesh.CARTESIAN)
    coords, kinds = _kinds(grid, bc)
    shape = tuple(c.size for c in coords)
    periodic = tuple(k[0] == mesh.PERIODIC and c.size > 1 for k, c in zip(kinds, coords))
    pinned = tuple((k[0] == mesh.DIRICHLET, k[1] == mesh.DIRICHLET) for k in kinds)
    info = [_axis_info(coords[a], periodic[a]) for a in range(3)]
    n0, n1, n2 = shape
    two, one = {}, {}
    wo = [{}, {}, {}]
    if metric == mesh.SPHERICAL:
        _spherical_tables(coords, kinds, periodic, info, two, one, wo)
    else:
        if any(mesh.AXIS in k for k in kinds):
            raise ValueError("the 'axis' boundary kind needs a spherical grid")
        _cartesian_tables(coords, periodic, info, two, one, wo)
    one["igv"] = 1.0 / one["gv"]
    two["iV2"] = 1.0 / two["V2"]
    two["Val2"] = (wo[0]["+"] + wo[0]["-"])[:, None] * (wo[1]["+"] + wo[1]["-"])[None, :]
    one["Valg"] = wo[2]["+"] + wo[2]["-"]
    two["iVal2"] = 1.0 / two["Val2"]
    one["iValg"] = 1.0 / one["Valg"]
    for s0 in SIGNS:
        for s1 in SIGNS:
            two["wo01" + s0 + s1] = wo[0][s0][:, None] * wo[1][s1][None, :]
    for s in SIGNS:
        one["wo2" + s] = wo[2][s].copy()
    rot = _rotation_tables(coords, metric, n1)
    return GlobalTables(shape, metric == mesh.SPHERICAL, periodic, pinned, two, one, rot)


def _cartesian_tables(coords, periodic, info, two, one, wo):
    n0, n1, n2 = (c.size for c in coords)
    w = [_dual(coords[a], periodic[a]) for a in range(3)]
    ihp = [_inv_where(info[a][0], info[a][2]) for a in range(3)]
    two["W0"] = np.ascontiguousarray((w[1][None, :] * ihp[0][:, None]) * np.ones((n0, n1)))
    two["W1"] = np.ascontiguousarray((w[0][:, None] * ihp[1][None, :]) * np.ones((n0, n1)))
    two["W2"] = np.ascontiguousarray((w[0][:, None] * w[1][None, :]) * np.ones((n0, n1)))
    one["g0"] = w[2].copy()
    one["g1"] = w[2].copy()
    one["g2"] = ihp[2]
    two["V2"] = w[0][:, None] * w[1][None, :]
    one["gv"] = w[2].copy()
    ones2 = np.ones((n0, n1))
    ones1 = np.ones(n2)
    for a in range(3):
        hp, hm, okp, okm = info[a]
        if coords[a].size > 1:
            wo[a]["+"] = np.where(okp, 0.5 * hp, 0.0)
            wo[a]["-"] = np.where(okm, 0.5 * hm, 0.0)
        else:
            wo[a]["+"] = np.full(coords[a].size, 0.5)
            wo[a]["-"] = np.full(coords[a].size, 0.5)
        for s, (h, ok) in (("+", (hp, okp)), ("-", (hm, okm))):
            inv = _inv_where(h, ok)
            key = f"{a}{s}"
            if a == 0:
                two["iL2_" + key] = inv[:, None] * ones2
                one["iL1_" + key] = ones1.copy()
            elif a == 1:
                two["iL2_" + key] = inv[None, :] * ones2
                one["iL1_" + key] = ones1.copy()
            else:
                two["iL2_" + key] = ones2.copy()
                one["iL1_" + key] = inv


def _spherical_tables(coords, kinds, periodic, info, two, one, wo):
    r, th, ph = coords
    n0, n1, n2 = r.size, th.size, ph.size
    if kinds[1] != (mesh.AXIS, mesh.AXIS):
        raise ValueError("spherical grids need the 'axis' kind on both theta faces")
    if not periodic[2]:
        raise ValueError("spherical grids need a periodic phi axis")
    if mesh.PERIODIC in kinds[0]:
        raise ValueError("r cannot be periodic")
    dph = np.diff(ph)
    if not np.allclose(dph, dph[0], rtol=1e-12, atol=0.0) or not math.isclose(
            ph[-1] - ph[0] + dph[0], 2.0 * math.pi, rel_tol=1e-12):
        raise ValueError("spherical phi must be uniform and cover [0, 2 pi)")
    mid = 0.5 * (r[:-1] + r[1:])
    rp = np.concatenate([mid, r[-1:]])
    rm = np.concatenate([r[:1], mid])
    drd = rp - rm
    Vr = (rp * rp * rp - rm * rm * rm) / 3.0
    tmid = 0.5 * (th[:-1] + th[1:])
    tp = np.concatenate([tmid, [math.pi]])
    tm = np.concatenate([[0.0], tmid])
    St = _cos(tm) - _cos(tp)
    dth = th[1:] - th[:-1]
    hp0, hm0, okp0, okm0 = info[0]
    # phi: the exact uniform spacing 2 pi / n2 (the
    # differences of the coordinates 2 pi k / n2 wander in the last bit), so
    # every phi metric factor is one constant -- the TMA march folds them into
    # its per-(r, theta) row records (oracle/geometry.py does the same)
    h2 = 2.0 * math.pi / n2
    hp2 = np.full(n2, h2)
    hm2 = np.full(n2, h2)
    okp2 = np.ones(n2, bool)
    okm2 = np.ones(n2, bool)
    wphi = np.full(n2, h2)
    W0 = ((rp * rp)[:, None] * St[None, :]) * _inv_where(hp0, okp0)[:, None]
    W0[-1, :] = 0.0
    W1 = np.zeros((n0, n1))
    W1[:, :-1] = (drd[:, None] * _sin(tmid)[None, :]) / dth[None, :]
    two["W0"] = np.ascontiguousarray(W0)
    two["W1"] = W1
    two["W2"] = (drd[:, None] * (tp - tm)[None, :]) / _sin(th)[None, :]
    one["g0"] = wphi.copy()
    one["g1"] = wphi.copy()
    one["g2"] = _inv_where(hp2, okp2)
    two["V2"] = Vr[:, None] * St[None, :]
    one["gv"] = wphi.copy()
    r3 = r * r * r
    d6 = (r3[1:] - r3[:-1]) / 6.0
    wo[0]["+"] = np.concatenate([d6, [0.0]])
    wo[0]["-"] = np.concatenate([[0.0], d6])
    ct = _cos(th)
    c2 = (ct[:-1] - ct[1:]) / 2.0
    wo[1]["+"] = np.concatenate([c2, [0.0]])
    wo[1]["-"] = np.concatenate([[0.0], c2])
    wo[2]["+"] = np.where(okp2, 0.5 * hp2, 0.0)
    wo[2]["-"] = np.where(okm2, 0.5 * hm2, 0.0)
    ones2 = np.ones((n0, n1))
    ones1 = np.ones(n2)
    two["iL2_0+"] = _inv_where(hp0, okp0)[:, None] * ones2
    two["iL2_0-"] = _inv_where(hm0, okm0)[:, None] * ones2
    one["iL1_0+"] = ones1.copy()
    one["iL1_0-"] = ones1.copy()
    dtp = np.concatenate([dth, [0.0]])
    dtm = np.concatenate([[0.0], dth])
    Ltp = r[:, None] * dtp[None, :]
    Ltm = r[:, None] * dtm[None, :]
    two["iL2_1+"] = _inv_where(Ltp, Ltp > 0)
    two["iL2_1-"] = _inv_where(Ltm, Ltm > 0)
    one["iL1_1+"] = ones1.copy()
    one["iL1_1-"] = ones1.copy()
    Lp = r[:, None] * _sin(th)[None, :]
    two["iL2_2+"] = 1.0 / Lp
    two["iL2_2-"] = 1.0 / Lp
    one["iL1_2+"] = _inv_where(hp2, okp2)
    one["iL1_2-"] = _inv_where(hm2, okm2)


def _frame(theta, phi):
    st, ct, sp, cp = math.sin(theta), math.cos(theta), math.sin(phi), math.cos(phi)
    return ((st * cp, st * sp, ct), (ct * cp, ct * sp, -st), (-sp, cp, 0.0))


def _rotation_tables(coords, metric, n1):
    rot = {}
    th = coords[1]
    dph = coords[2][1] - coords[2][0] if coords[2].size > 1 else 0.0
    for f in FACES:
        M = np.zeros((n1, 3, 3))
        for j in range(n1):
            edge = (f == "t+" and j + 1 >= n1) or (f == "t-" and j == 0)
            if metric != mesh.SPHERICAL or edge:
                M[j] = np.eye(3)
                continue
            Rc = _frame(th[j], 0.0)
            Rn = {"t+": lambda: _frame(th[j + 1], 0.0), "t-": lambda: _frame(th[j - 1], 0.0),
                  "p+": lambda: _frame(th[j], dph), "p-": lambda: _frame(th[j], -dph)}[f]()
            for a in range(3):
                for b in range(3):
                    M[j, a, b] = (Rc[a][0] * Rn[b][0] + Rc[a][1] * Rn[b][1]) + Rc[a][2] * Rn[b][2]
        A = np.abs(M)
        rot["M" + f] = M.reshape(n1, 9)
        rot["R" + f] = (1.0 + ((A[:, :, 0] + A[:, :, 1]) + A[:, :, 2])) if metric == mesh.SPHERICAL else np.full((n1, 3), 2.0)
    return rot


TWO_ORDER_1 = ["W0", "W1", "W2"]
ONE_ORDER_1 = ["g0", "g1", "g2"]


def pack(gt: GlobalTables, i0: int = 0, n0_local: int | None = None, ghost_lo=False, ghost_hi=False, phi=None):
    """Flat table array for the axis-0 slab [i0, i0 + n0_local), ghost rows
    filled from the global tables when the neighbour slab exists.
    ``phi = (k0, n)``: a phi-slab -- the columns [k0, k0 + n) plus one ghost
    column on each side (the neighbours' columns, periodically); the ghost
    columns carry zero inner-product weight (gv = Valg = 0: never summed) and
    are pinned by flags() (never advanced)."""
    n0, n1, n2 = gt.shape
    if n0_local is None:
        n0_local = n0
    cols = None
    if phi is not None:
        k0, nl = phi
        cols = np.array([(k0 - 1 + c) % n2 for c in range(nl + 2)])

    def two(name):
        t = gt.two[name]
        out = np.zeros((n0_local + 2, n1))
        out[1:-1] = t[i0:i0 + n0_local]
        if ghost_lo:
            out[0] = t[(i0 - 1) % n0]
        if ghost_hi:
            out[-1] = t[(i0 + n0_local) % n0]
        return out.ravel()

    def one(name):
        t = np.asarray(gt.one[name], float).ravel()
        if cols is None:
            return t
        t = t[cols].copy()
        if name in ("gv", "Valg"):  # ghost columns: zero weight
            t[0] = 0.0
            t[-1] = 0.0
        return t

    parts = [two(n) for n in TWO_ORDER_1] + [one(n) for n in ONE_ORDER_1]
    parts += [two("iV2"), one("igv")]
    parts += [two(f"iL2_{a}{s}") for a in range(3) for s in SIGNS]
    parts += [one(f"iL1_{a}{s}") for a in range(3) for s in SIGNS]
    parts += [two("wo01" + s0 + s1) for s0 in SIGNS for s1 in SIGNS]
    parts += [one("wo2" + s) for s in SIGNS]
    parts += [two("iVal2"), one("iValg")]
    parts += [gt.rot["M" + f].ravel() for f in FACES]
    parts += [gt.rot["R" + f].ravel() for f in FACES]
    parts += [two("V2"), one("gv"), two("Val2"), one("Valg")]
    return np.ascontiguousarray(np.concatenate(parts))


def flags(gt: GlobalTables, i0=0, n0_local=None, ghost_lo=False, ghost_hi=False, phi=None):
    n0 = gt.shape[0]
    if n0_local is None:
        n0_local = n0
    f = np.zeros(NFLAGS, dtype=np.int32)
    f[0:3] = [int(p) for p in gt.periodic]
    f[3:9] = [int(x) for pair in gt.pinned for x in pair]
    # a slab only pins the global axis-0 ends; the kernel tests global indices
    f[9] = int(ghost_lo)
    f[10] = int(ghost_hi)
    f[11] = n0
    f[12] = i0
    f[13] = int(gt.spherical)
    f[15] = gt.shape[2]
    if phi is not None:  # phi-slab: periodic phi, ghost columns 0 and n + 1 pinned
        if not gt.periodic[2]:
            raise ValueError("phi-slabs need a periodic axis 2")
        f[2] = 1
        f[7] = 1
        f[8] = 1
        f[14] = 1
        f[16] = phi[0]
    return f


def slab_bounds(n0: int, nranks: int, rank: int):
    """Balanced axis-0 (r) slabs: the first n0 % nranks ranks get one extra plane."""
    base, extra = divmod(n0, nranks)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return start, count
