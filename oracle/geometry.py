"""Oracle metric tables (test infrastructure; see oracle/__init__.py).

Restates the discretisation geometry of the reference path:

* node-centred tensor-product grid, one ghost layer, Dirichlet nodes pinned,
  periodic wrap spacing = mean of the two edge spacings, half dual cells at
  non-periodic ends -- reference ``mesh.py:1-15``, ``mesh.py:130-156``
  (``Grid.wrap_spacing``, ``Grid.dual_widths``, ``Grid.dual_volumes``);
* spherical (r, theta, phi) extension (parity unpinned):
  r node-centred with half cells at the ends, theta cell-centred on (0, pi)
  with zero-area faces at the poles ("axis" boundary), phi uniform periodic.

Everything is embedded in three axes: a 1-D or 2-D reference grid gets
trailing singleton axes that carry no faces and no neighbours.

All tables are separable: a 2-D part over (axis0, axis1) times a 1-D part
over axis2, so a cell quantity is ``T2[i, j] * t1[k]`` evaluated in exactly
that order by both the oracle and the CUDA kernels.
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math

import numpy as np

DIRICHLET = "dirichlet"
NEUMANN = "neumann"
PERIODIC = "periodic"
AXIS = "axis"
NONE = "none"  # singleton padding axis


@dataclass
class OracleGeometry:
    shape: tuple
    metric: str
    kinds: tuple  # ((lo, hi),) * 3
    periodic: tuple
    real: tuple  # axis has >1 node
    # scalar 7-point finite-volume tables
    W2: list = field(default_factory=list)  # W2[a] : (n0, n1) face (+ side) weight 2-D part
    g1: list = field(default_factory=list)  # g1[a] : (n2,) face weight 1-D part
    iV2: np.ndarray = None
    igv: np.ndarray = None
    V2: np.ndarray = None
    gv: np.ndarray = None
    # aligned (19-point) tables
    iL2: dict = field(default_factory=dict)  # (a, s) -> (n0, n1)
    iL1: dict = field(default_factory=dict)  # (a, s) -> (n2,)
    wo01: dict = field(default_factory=dict)  # (s0, s1) -> (n0, n1)
    wo2: dict = field(default_factory=dict)  # s2 -> (n2,)
    iVal2: np.ndarray = None
    iValg: np.ndarray = None
    Val2: np.ndarray = None
    Valg: np.ndarray = None
    # spherical vector rotation tables: face -> (n1, 3, 3); rowabs -> (n1, 3)
    M: dict = field(default_factory=dict)
    Rabs: dict = field(default_factory=dict)

    @property
    def pinned(self) -> np.ndarray:
        """mesh.pinned_mask (mesh.py:311-324) embedded in 3 axes."""
        m = np.zeros(self.shape, dtype=bool)
        for a in range(3):
            lo, hi = self.kinds[a]
            sl = [slice(None)] * 3
            if lo == DIRICHLET:
                sl[a] = 0
                m[tuple(sl)] = True
            if hi == DIRICHLET:
                sl[a] = self.shape[a] - 1
                m[tuple(sl)] = True
        return m

    def volume(self) -> np.ndarray:
        """Scalar finite-volume control volume per node (n0, n1, n2)."""
        return self.V2[:, :, None] * self.gv[None, None, :]

    def aligned_volume(self) -> np.ndarray:
        return self.Val2[:, :, None] * self.Valg[None, None, :]


def _spacings(x: np.ndarray, periodic: bool):
    """next-spacing h[i] = x[i+1]-x[i] (wrap spacing at the seam if periodic,
    mesh.py:130-133), and whether each +/- neighbour exists."""
    n = x.size
    h = np.zeros(n)
    if n > 1:
        h[:-1] = x[1:] - x[:-1]
        if periodic:
            h[-1] = 0.5 * (h[0] + h[-2])
    hp = h.copy()  # spacing to +neighbour
    hm = np.zeros(n)
    if n > 1:
        hm[1:] = h[:-1]
        if periodic:
            hm[0] = h[-1]
    has_p = np.zeros(n, dtype=bool)
    has_m = np.zeros(n, dtype=bool)
    if n > 1:
        has_p[:-1] = True
        has_m[1:] = True
        if periodic:
            has_p[-1] = True
            has_m[0] = True
    hp = np.where(has_p, hp, 0.0)
    hm = np.where(has_m, hm, 0.0)
    return hp, hm, has_p, has_m


def _dual_widths(x: np.ndarray, periodic: bool) -> np.ndarray:
    """mesh.Grid.dual_widths (mesh.py:135-149); singleton axis -> 1."""
    n = x.size
    if n == 1:
        return np.ones(1)
    h = x[1:] - x[:-1]
    w = np.empty(n)
    w[1:-1] = 0.5 * (h[:-1] + h[1:])
    if periodic:
        hw = 0.5 * (h[0] + h[-1])
        w[0] = 0.5 * (hw + h[0])
        w[-1] = 0.5 * (h[-1] + hw)
    else:
        w[0] = 0.5 * h[0]
        w[-1] = 0.5 * h[-1]
    return w


def _safe_inv(h: np.ndarray, ok: np.ndarray) -> np.ndarray:
    out = np.zeros_like(h)
    out[ok] = 1.0 / h[ok]
    return out


def build_geometry(coords, kinds, metric: str = "cartesian") -> OracleGeometry:
    """coords: list of 1..3 node arrays; kinds: list of (lo, hi) kind strings."""
    coords = [np.asarray(c, dtype=float) for c in coords]
    kinds = [tuple(k) for k in kinds]
    while len(coords) < 3:
        coords.append(np.zeros(1))
        kinds.append((NONE, NONE))
    shape = tuple(c.size for c in coords)
    periodic = tuple(k[0] == PERIODIC and c.size > 1 for k, c in zip(kinds, coords))
    real = tuple(c.size > 1 for c in coords)
    g = OracleGeometry(shape=shape, metric=metric, kinds=tuple(kinds), periodic=periodic, real=real)
    n0, n1, n2 = shape
    sp = [_spacings(coords[a], periodic[a]) for a in range(3)]
    if metric == "cartesian":
        _cartesian(g, coords, sp)
    elif metric == "spherical":
        _spherical(g, coords, sp)
    else:
        raise ValueError(f"unknown metric {metric!r}")
    g.iV2 = 1.0 / g.V2
    g.igv = 1.0 / g.gv
    g.Val2 = _wsum(g, 0)[:, None] * _wsum(g, 1)[None, :]
    g.Valg = g.wo2["+"] + g.wo2["-"]
    g.iVal2 = 1.0 / g.Val2
    g.iValg = 1.0 / g.Valg
    return g


def _wsum(g, a):
    return g._wo[a]["+"] + g._wo[a]["-"]


def _cartesian(g, coords, sp):
    n0, n1, n2 = g.shape
    w = [_dual_widths(coords[a], g.periodic[a]) for a in range(3)]
    # scalar FV: face (+ side of node) weights = transverse dual area / spacing
    W = []
    for a in range(3):
        hp, hm, has_p, has_m = sp[a]
        ihp = _safe_inv(hp, has_p)
        if a == 0:
            W.append(w[1][None, :] * ihp[:, None])
        elif a == 1:
            W.append(w[0][:, None] * ihp[None, :])
        else:
            W.append(w[0][:, None] * w[1][None, :])
    g.W2 = [np.ascontiguousarray(x * np.ones((n0, n1))) for x in W]
    hp2, hm2, hasp2, hasm2 = sp[2]
    g.g1 = [w[2].copy(), w[2].copy(), _safe_inv(hp2, hasp2)]
    g.V2 = w[0][:, None] * w[1][None, :]
    g.gv = w[2].copy()
    # aligned: inverse one-sided edge lengths and octant weights
    ones2 = np.ones((n0, n1))
    ones1 = np.ones(n2)
    wo = []
    for a in range(3):
        hp, hm, has_p, has_m = sp[a]
        d = {}
        if g.real[a]:
            d["+"] = np.where(has_p, 0.5 * hp, 0.0)
            d["-"] = np.where(has_m, 0.5 * hm, 0.0)
        else:
            d["+"] = np.full(coords[a].size, 0.5)
            d["-"] = np.full(coords[a].size, 0.5)
        wo.append(d)
        for s, (hh, ok) in (("+", (hp, has_p)), ("-", (hm, has_m))):
            inv = _safe_inv(hh, ok)
            if a == 0:
                g.iL2[(a, s)] = inv[:, None] * ones2
                g.iL1[(a, s)] = ones1.copy()
            elif a == 1:
                g.iL2[(a, s)] = inv[None, :] * ones2
                g.iL1[(a, s)] = ones1.copy()
            else:
                g.iL2[(a, s)] = ones2.copy()
                g.iL1[(a, s)] = inv
    g._wo = wo
    for s0 in "+-":
        for s1 in "+-":
            g.wo01[(s0, s1)] = wo[0][s0][:, None] * wo[1][s1][None, :]
    g.wo2 = {s: wo[2][s].copy() for s in "+-"}
    for f in ("t+", "t-", "p+", "p-"):
        g.M[f] = np.broadcast_to(np.eye(3), (n1, 3, 3)).copy()
        g.Rabs[f] = np.full((n1, 3), 2.0)


def _msin(x):
    """Scalar libm sin per element (independent of numpy's SIMD dispatch)."""
    return np.array([math.sin(v) for v in np.ravel(x)]).reshape(np.shape(x))


def _mcos(x):
    return np.array([math.cos(v) for v in np.ravel(x)]).reshape(np.shape(x))


def _frame(theta, phi):
    st, ct, sp_, cp = math.sin(theta), math.cos(theta), math.sin(phi), math.cos(phi)
    er = (st * cp, st * sp_, ct)
    et = (ct * cp, ct * sp_, -st)
    ep = (-sp_, cp, 0.0)
    return (er, et, ep)  # rows = local unit vectors


def _rel_rotation(Rc, Rn):
    """M[a][b] = e_a(centre) . e_b(neighbour), summed in index order."""
    M = np.empty((3, 3))
    for a in range(3):
        for b in range(3):
            M[a, b] = (Rc[a][0] * Rn[b][0] + Rc[a][1] * Rn[b][1]) + Rc[a][2] * Rn[b][2]
    return M


def _spherical(g, coords, sp):
    r, th, ph = coords
    n0, n1, n2 = g.shape
    if g.kinds[1] != (AXIS, AXIS):
        raise ValueError("spherical grids need the 'axis' kind on both theta faces")
    if not g.periodic[2]:
        raise ValueError("spherical grids need a periodic phi axis")
    if not (th[0] > 0.0 and th[-1] < math.pi):
        raise ValueError("theta nodes must lie strictly inside (0, pi)")
    if g.kinds[0][0] == PERIODIC:
        raise ValueError("r cannot be periodic")
    # r: node-centred faces with half cells at the ends
    rf = 0.5 * (r[:-1] + r[1:])
    rp = np.empty(n0)
    rm = np.empty(n0)
    rp[:-1] = rf
    rp[-1] = r[-1]
    rm[1:] = rf
    rm[0] = r[0]
    drd = rp - rm
    Vr = (rp * rp * rp - rm * rm * rm) / 3.0
    # theta: cell-centred, pole faces at 0 and pi
    tf = 0.5 * (th[:-1] + th[1:])
    tp = np.empty(n1)
    tm = np.empty(n1)
    tp[:-1] = tf
    tp[-1] = math.pi
    tm[1:] = tf
    tm[0] = 0.0
    St = _mcos(tm) - _mcos(tp)
    dth = th[1:] - th[:-1]
    # phi: the exact uniform spacing 2 pi / n2 (DESIGN.md §2 D1: constant phi
    # metric factors; the coordinate differences wander in the last bit)
    h2 = 2.0 * math.pi / n2
    hp2, hm2 = np.full(n2, h2), np.full(n2, h2)
    hasp2, hasm2 = np.ones(n2, bool), np.ones(n2, bool)
    wphi = np.full(n2, h2)
    h0p, h0m, has0p, has0m = sp[0]
    ih0p = _safe_inv(h0p, has0p)
    W0 = ((rp * rp)[:, None] * St[None, :]) * ih0p[:, None]
    W0[-1, :] = 0.0
    W1 = np.zeros((n0, n1))
    W1[:, :-1] = (drd[:, None] * _msin(tf)[None, :]) / dth[None, :]
    W2 = (drd[:, None] * (tp - tm)[None, :]) / _msin(th)[None, :]
    g.W2 = [np.ascontiguousarray(W0), W1, W2]
    g.g1 = [wphi.copy(), wphi.copy(), _safe_inv(hp2, hasp2)]
    g.V2 = Vr[:, None] * St[None, :]
    g.gv = wphi.copy()
    # aligned tables
    ones1 = np.ones(n2)
    r3 = r * r * r
    wo0 = {"+": np.zeros(n0), "-": np.zeros(n0)}
    wo0["+"][:-1] = (r3[1:] - r3[:-1]) / 6.0
    wo0["-"][1:] = (r3[1:] - r3[:-1]) / 6.0
    ct = _mcos(th)
    wo1 = {"+": np.zeros(n1), "-": np.zeros(n1)}
    wo1["+"][:-1] = (ct[:-1] - ct[1:]) / 2.0
    wo1["-"][1:] = (ct[:-1] - ct[1:]) / 2.0
    wo2 = {"+": np.where(hasp2, 0.5 * hp2, 0.0), "-": np.where(hasm2, 0.5 * hm2, 0.0)}
    g._wo = [wo0, wo1, wo2]
    for s0 in "+-":
        for s1 in "+-":
            g.wo01[(s0, s1)] = wo0[s0][:, None] * wo1[s1][None, :]
    g.wo2 = {s: wo2[s].copy() for s in "+-"}
    ir0p = _safe_inv(h0p, has0p)
    ir0m = _safe_inv(h0m, has0m)
    ones2 = np.ones((n0, n1))
    g.iL2[(0, "+")] = ir0p[:, None] * ones2
    g.iL2[(0, "-")] = ir0m[:, None] * ones2
    g.iL1[(0, "+")] = ones1.copy()
    g.iL1[(0, "-")] = ones1.copy()
    dtp = np.zeros(n1)
    dtm = np.zeros(n1)
    dtp[:-1] = dth
    dtm[1:] = dth
    Ltp = r[:, None] * dtp[None, :]
    Ltm = r[:, None] * dtm[None, :]
    g.iL2[(1, "+")] = _safe_inv(Ltp, Ltp > 0)
    g.iL2[(1, "-")] = _safe_inv(Ltm, Ltm > 0)
    g.iL1[(1, "+")] = ones1.copy()
    g.iL1[(1, "-")] = ones1.copy()
    Lp = r[:, None] * _msin(th)[None, :]
    g.iL2[(2, "+")] = 1.0 / Lp
    g.iL2[(2, "-")] = 1.0 / Lp
    g.iL1[(2, "+")] = _safe_inv(hp2, hasp2)
    g.iL1[(2, "-")] = _safe_inv(hm2, hasm2)
    # vector-viscosity relative rotations M = R_c R_nb^T
    dph = ph[1] - ph[0]
    for f in ("t+", "t-", "p+", "p-"):
        M = np.zeros((n1, 3, 3))
        for j in range(n1):
            Rc = _frame(th[j], 0.0)
            if (f == "t+" and j + 1 >= n1) or (f == "t-" and j == 0):
                M[j] = np.eye(3)  # no neighbour across the pole
                continue
            if f == "t+":
                Rn = _frame(th[j + 1], 0.0)
            elif f == "t-":
                Rn = _frame(th[j - 1], 0.0)
            elif f == "p+":
                Rn = _frame(th[j], dph)
            else:
                Rn = _frame(th[j], -dph)
            M[j] = _rel_rotation(Rc, Rn)
        g.M[f] = M
        A = np.abs(M)
        g.Rabs[f] = 1.0 + ((A[:, :, 0] + A[:, :, 1]) + A[:, :, 2])
