"""Oracle right-hand sides F(u) and explicit-Euler limits (test infrastructure).

Restates SPEC.md ``operators``:

* ``scalar_apply``   -- F = (1/rho) div(nu rho grad u), conservative flux
  difference with ARITHMETIC face average of nu*rho, divided by rho at the
  node; component-wise for multi-component fields
  (SPEC.md:108).  With ``vector_metric`` on a spherical grid the components
  (v_r, v_theta, v_phi) are rotated into the centre cell's frame before
  differencing (the vector Laplacian's metric terms).
* ``aligned_apply``  -- F = pref/rho div(c b b . grad T), c = f_c f_m(T0)
  kappa0 T0^{5/2} evaluated at nodes.  The
  symmetric 19-point discretisation is the gradient of the quadratic form
  Q = 1/2 sum_{v,sigma} W_{v,sigma} (beta_v . g_{v,sigma})^2, beta = sqrt(c) b
  (so c_v (b_v . g)^2 = (beta_v . g)^2), over the 8
  one-sided "corner tetrahedra" of every node: symmetric in the rho*V inner
  product, negative semi-definite, and identical to the scalar stencil with
  arithmetic face-averaged c when b is axis-aligned in 1-D.
* ``*_gershgorin``   -- Delta t_Euler = 2 / max_i sum_j |J_ij| over
  non-pinned rows.

Pinned (Dirichlet) nodes get F = 0 (mesh.py:5-7).  Arrays are SoA
(ncomp, n0, n1, n2).  Operation order is explicit and mirrored by the CUDA
kernels (see csrc/ops_*.cuh).
"""
from __future__ import annotations

import numpy as np

SIG = [(s0, s1, s2) for s0 in "+-" for s1 in "+-" for s2 in "+-"]  # canonical order


def shift(x, axis, d, periodic):
    """y[i] = x[i+d] along ``axis`` (last 3 dims); wraps if periodic, else the
    node itself at the edge (so a difference across a missing face is 0)."""
    ax = x.ndim - 3 + axis
    n = x.shape[ax]
    if n == 1:
        return x
    if periodic:
        return np.roll(x, -d, axis=ax)
    y = np.roll(x, -d, axis=ax)
    sl = [slice(None)] * x.ndim
    sl[ax] = n - 1 if d > 0 else 0
    y[tuple(sl)] = x[tuple(sl)]
    return y


def shift_zero(x, axis, d, periodic):
    """Like ``shift`` but 0 where the neighbour does not exist."""
    ax = x.ndim - 3 + axis
    n = x.shape[ax]
    if n == 1:
        return np.zeros_like(x)
    y = np.roll(x, -d, axis=ax)
    if not periodic:
        sl = [slice(None)] * x.ndim
        sl[ax] = n - 1 if d > 0 else 0
        y[tuple(sl)] = 0.0
    return y


def _b2(t):
    return t[:, :, None]


def _b1(t):
    return t[None, None, :]


def face_coefs(geom):
    """Per-node face coefficients W*g for the + and - faces of each axis."""
    out = []
    for a in range(3):
        cp = _b2(geom.W2[a]) * _b1(geom.g1[a])
        if a < 2:
            Wm = shift_zero(geom.W2[a][:, :, None] * np.ones((1, 1, geom.shape[2])), a, -1, geom.periodic[a])
            cm = Wm * _b1(geom.g1[a])
        else:
            gm = np.roll(geom.g1[2], 1) if geom.periodic[2] else np.concatenate([[0.0], geom.g1[2][:-1]])
            if geom.shape[2] == 1:
                gm = np.zeros(1)
            cm = _b2(geom.W2[2]) * _b1(gm)
        out.append((cm, cp))
    return out


def _dface(D, a, d, periodic):
    if D is None:
        return None
    if np.isscalar(D):
        return D
    return 0.5 * (D + shift(D, a, d, periodic))


def scalar_apply(geom, u, D=None, rho=None, vector_metric=False):
    """F(u) for the scalar (or component-wise / vector) diffusion operator.

    u: (ncomp, n0, n1, n2).  D = nu*rho nodal (None == 1), rho nodal or None.
    Face term: t = (Dface * (W*g)) * (u_nb - u_c); sum order
    ((((t0m + t0p) + t1m) + t1p) + t2m) + t2p; F = (S * iv) * (1 / rho).
    """
    ncomp = u.shape[0]
    per = geom.periodic
    coefs = face_coefs(geom)
    iv = _b2(geom.iV2) * _b1(geom.igv)
    irho = None if rho is None else 1.0 / rho  # (1/rho) div(...): one reciprocal per node
    rot = vector_metric and geom.metric == "spherical" and ncomp == 3
    F = np.empty_like(u)
    nbs = {}
    for a in range(3):
        for d, tag in ((-1, "m"), (1, "p")):
            nbs[(a, tag)] = shift(u, a, d, per[a])
    for c in range(ncomp):
        S = None
        for a in range(3):
            for tag, idx in (("m", 0), ("p", 1)):
                coef = coefs[a][idx]
                nb = nbs[(a, tag)]
                if rot and a > 0:
                    M = geom.M[("t" if a == 1 else "p") + ("+" if tag == "p" else "-")]
                    Mc = M[:, c, :]  # (n1, 3)
                    m0 = Mc[None, :, 0, None]
                    m1 = Mc[None, :, 1, None]
                    m2 = Mc[None, :, 2, None]
                    val = ((m0 * nb[0]) + (m1 * nb[1])) + (m2 * nb[2])
                else:
                    val = nb[c]
                du = val - u[c]
                Df = _dface(D, a, -1 if tag == "m" else 1, per[a])
                if Df is None:
                    t = coef * du
                else:
                    t = (Df * coef) * du
                S = t if S is None else S + t
        Fc = S * iv
        if irho is not None:
            Fc = Fc * irho
        F[c] = Fc
    F[:, geom.pinned] = 0.0
    return F


def scalar_row_terms(geom, D=None):
    """Per-node sum of face coefficients in the canonical order (no abs
    needed: every face coefficient is >= 0)."""
    coefs = face_coefs(geom)
    per = geom.periodic
    S = None
    for a in range(3):
        for tag, idx in (("m", 0), ("p", 1)):
            Df = _dface(D, a, -1 if tag == "m" else 1, per[a])
            t = coefs[a][idx] if Df is None else Df * coefs[a][idx]
            S = t if S is None else S + t
    return S


def scalar_gershgorin(geom, D=None, rho=None, ncomp=1, vector_metric=False):
    """Row bound lam_i = sum_j |J_ij| per node and component.

    scalar: (sum_f c_f * 2) * iv / rho.  vector: sum_f c_f * R_f[a] with
    R = 2 for r faces and 1 + sum_b |M_f[a][b]| for theta/phi faces.
    Returns lam (ncomp, n0, n1, n2) with pinned rows zeroed.
    """
    coefs = face_coefs(geom)
    per = geom.periodic
    iv = _b2(geom.iV2) * _b1(geom.igv)
    rot = vector_metric and geom.metric == "spherical" and ncomp == 3
    lam = np.empty((ncomp,) + geom.shape)
    for c in range(ncomp):
        S = None
        for a in range(3):
            for tag, idx in (("m", 0), ("p", 1)):
                Df = _dface(D, a, -1 if tag == "m" else 1, per[a])
                t = coefs[a][idx] if Df is None else Df * coefs[a][idx]
                if rot and a > 0:
                    R = geom.Rabs[("t" if a == 1 else "p") + ("+" if tag == "p" else "-")][:, c]
                    t = t * R[None, :, None]
                else:
                    t = t * 2.0
                S = t if S is None else S + t
        L = S * iv
        if rho is not None:
            L = L / rho
        lam[c] = L
    lam[:, geom.pinned] = 0.0
    return lam


def scalar_diag(geom, D=None, rho=None):
    """-J_ii (>= 0) for the Jacobi preconditioner: (sum_f c_f) * iv / rho."""
    S = scalar_row_terms(geom, D)
    d = S * (_b2(geom.iV2) * _b1(geom.igv))
    if rho is not None:
        d = d / rho
    d = d.copy()
    d[geom.pinned] = 0.0
    return d


def euler_dt(lam):
    m = float(np.max(lam)) if lam.size else 0.0
    if not m > 0.0:
        return float("inf")
    return 2.0 / m


# --------------------------------------------------------------------------
# field-aligned (Spitzer) conduction
# --------------------------------------------------------------------------

def aligned_coefficient(T0, kappa0=1.0, fc=None, T_floor=1e-10):
    """c = ((kappa0 * f_c(r)) * f_m) * ((T0f*T0f) * sqrt(T0f)), T0f = max(T0, T_floor)
    (SPEC.md:117-119, :144-145).  ``fc`` is a per-axis0 table or None (== 1);
    f_m is the constant 1 preset."""
    if np.any(~(T0 > 0.0)):
        raise ValueError("aligned conduction: non-positive T0 (domain error, SPEC.md:120)")
    T0f = np.maximum(T0, T_floor)
    p = (T0f * T0f) * np.sqrt(T0f)
    k = np.full(T0.shape[0], float(kappa0)) if fc is None else float(kappa0) * np.asarray(fc, float)
    return k[:, None, None] * p


def _iL(geom, a, s):
    return _b2(geom.iL2[(a, s)]) * _b1(geom.iL1[(a, s)])


def aligned_beta(b, c):
    """beta_a = b_a * sqrt(c): c b b^T = beta beta^T, so the frozen operator
    needs three nodal arrays instead of four ("Spitzer stencil")."""
    return b * np.sqrt(c)[None]


def aligned_E(geom, T, beta):
    """Per-node edge fluxes E[(a, s)] of the corner-tetrahedron quadratic form.

    bil[(a,s)] = beta_a * (iL2 * iL1); p = bil * dT (one-sided difference);
    f_sigma = (wo01 * wo2) * ((p_0 + p_1) + p_2); E = bil * sum_sigma f_sigma
    (octants in canonical order)."""
    per = geom.periodic
    p = {}
    bil = {}
    for a in range(3):
        Tp = shift(T, a, 1, per[a])
        Tm = shift(T, a, -1, per[a])
        bil[(a, "+")] = beta[a] * _iL(geom, a, "+")
        bil[(a, "-")] = beta[a] * _iL(geom, a, "-")
        p[(a, "+")] = bil[(a, "+")] * (Tp - T)
        p[(a, "-")] = bil[(a, "-")] * (T - Tm)
    f = {}
    for sg in SIG:
        s = (p[(0, sg[0])] + p[(1, sg[1])]) + p[(2, sg[2])]
        om = _b2(geom.wo01[(sg[0], sg[1])]) * _b1(geom.wo2[sg[2]])
        f[sg] = om * s
    E = {}
    for a in range(3):
        for s in "+-":
            acc = None
            for sg in SIG:
                if sg[a] == s:
                    acc = f[sg] if acc is None else acc + f[sg]
            E[(a, s)] = bil[(a, s)] * acc
    return E


def aligned_apply(geom, T, b, c, rho=None, pref=1.0):
    """F(T) = (G * iVal) * (0 - pref / rho), G = dQ/dT (see module docstring).

    T: (n0, n1, n2); b: (3, n0, n1, n2); c: (n0, n1, n2) nodal conductivity.
    G is summed in the order an r-marching kernel produces it:
      own = ((E0- - E0+) + (E1- - E1+)) + (E2- - E2+)          at the node
      nbr = (E1+(j-1) - E1-(j+1)) + (E2+(k-1) - E2-(k+1))     in-plane neighbours
      G   = (E0+(i-1) - E0-(i+1)) + (own + nbr)
    with missing neighbours contributing 0.
    """
    per = geom.periodic
    E = aligned_E(geom, T, aligned_beta(b, c))
    own = ((E[(0, "-")] - E[(0, "+")]) + (E[(1, "-")] - E[(1, "+")])) + (E[(2, "-")] - E[(2, "+")])
    nbr = (shift_zero(E[(1, "+")], 1, -1, per[1]) - shift_zero(E[(1, "-")], 1, 1, per[1])) + (
        shift_zero(E[(2, "+")], 2, -1, per[2]) - shift_zero(E[(2, "-")], 2, 1, per[2]))
    G = (shift_zero(E[(0, "+")], 0, -1, per[0]) - shift_zero(E[(0, "-")], 0, 1, per[0])) + (own + nbr)
    iv = _b2(geom.iVal2) * _b1(geom.iValg)
    # prefactor and density as one scale 0 - pref / rho (SPEC.md:117 F = pref/rho div(...)):
    # one product per node on the device, the division once per plane for a radial rho
    nscale = (0.0 - pref) if rho is None else 0.0 - (pref / rho)
    F = (G * iv) * nscale
    F = F.copy()
    F[geom.pinned] = 0.0
    return F


# 19-point offsets in canonical order: centre, faces, face-diagonals
OFFSETS = [(0, 0, 0)]
for _a in range(3):
    for _d in (-1, 1):
        o = [0, 0, 0]
        o[_a] = _d
        OFFSETS.append(tuple(o))
for _a in range(3):
    for _b in range(_a + 1, 3):
        for _da in (-1, 1):
            for _db in (-1, 1):
                o = [0, 0, 0]
                o[_a] = _da
                o[_b] = _db
                OFFSETS.append(tuple(o))
OFF_INDEX = {o: n for n, o in enumerate(OFFSETS)}


def _sgn(s):
    return 1.0 if s == "+" else -1.0


def aligned_hessian_rows(geom, beta):
    """H[m, off] = d^2 Q / dT_m dT_{m+off} for the 19 offsets, accumulated per
    row in a fixed order: first the 8 tets with apex v = m (canonical sigma
    order: diagonal, then the three edge ends), then the 24 tets with v = m -
    sigma_a e_a (a = 0..2, sigma_a = +,-, other sigmas canonical: diagonal,
    the apex, then the other two edge ends)."""
    per = geom.periodic
    shape = geom.shape
    H = [np.zeros(shape) for _ in OFFSETS]
    # q[(a, s)] at every node v: sigma_a * (beta_a * iL_{a, s})
    q = {}
    for a in range(3):
        for s in "+-":
            q[(a, s)] = _sgn(s) * (beta[a] * _iL(geom, a, s))
    om = {}
    for sg in SIG:
        om[sg] = _b2(geom.wo01[(sg[0], sg[1])]) * _b1(geom.wo2[sg[2]]) * np.ones(geom.shape)
    # (A) apex tets
    for sg in SIG:
        qa = [q[(a, sg[a])] for a in range(3)]
        qs = (qa[0] + qa[1]) + qa[2]
        w = om[sg]
        H[0] += (w * qs) * qs
        for a in range(3):
            off = [0, 0, 0]
            off[a] = 1 if sg[a] == "+" else -1
            H[OFF_INDEX[tuple(off)]] += (w * (0.0 - qs)) * qa[a]
    # (B) end-point tets: v = m - sigma_a e_a; quantities evaluated at v
    for a in range(3):
        for sa in "+-":
            d = -1 if sa == "+" else 1  # v = m + d e_a
            for sg in SIG:
                if sg[a] != sa:
                    continue
                qv = [shift_zero(q[(bb, sg[bb])], a, d, per[a]) for bb in range(3)]
                wv = shift_zero(om[sg], a, d, per[a])
                qs = (qv[0] + qv[1]) + qv[2]
                qa_ = qv[a]
                H[0] += (wv * qa_) * qa_
                off = [0, 0, 0]
                off[a] = d
                H[OFF_INDEX[tuple(off)]] += (wv * qa_) * (0.0 - qs)
                for bb in range(3):
                    if bb == a:
                        continue
                    off = [0, 0, 0]
                    off[a] = d
                    off[bb] = 1 if sg[bb] == "+" else -1
                    H[OFF_INDEX[tuple(off)]] += (wv * qa_) * qv[bb]
    return H


def aligned_gershgorin(geom, b, c, rho=None, pref=1.0):
    """lam_m = ((sum_off |H[m, off]| * iVal) * pref) / rho over non-pinned rows,
    and the Jacobi diagonal -J_mm = ((H[m,0] * iVal) * pref) / rho."""
    H = aligned_hessian_rows(geom, aligned_beta(b, c))
    S = None
    for h in H:
        S = np.abs(h) if S is None else S + np.abs(h)
    iv = _b2(geom.iVal2) * _b1(geom.iValg)
    lam = (S * iv) * pref
    dg = (H[0] * iv) * pref
    if rho is not None:
        lam = lam / rho
        dg = dg / rho
    lam = lam.copy()
    dg = dg.copy()
    lam[geom.pinned] = 0.0
    dg[geom.pinned] = 0.0
    return lam, dg


# ---------------------------------------------------------------- line-r preconditioner
# (PC2 substitute: block Jacobi over r-lines.  The r-line block
# of -J is a principal submatrix of a W-symmetric positive semi-definite
# matrix and, for the 7- and 19-point stencils, exactly tridiagonal, so
# M = a + dt (line block of -J) is SPD and the Thomas algorithm needs no
# pivoting.)

def aligned_line_offdiag(geom, b, c, rho=None, pref=1.0):
    """-J_{i,i-1}, -J_{i,i+1} of the aligned operator: ((H[m, -+e_r] * iVal)
    * pref) / rho, pinned rows 0 (same expression order as the diagonal)."""
    H = aligned_hessian_rows(geom, aligned_beta(b, c))
    iv = _b2(geom.iVal2) * _b1(geom.iValg)
    out = []
    for off in ((-1, 0, 0), (1, 0, 0)):
        j = (H[OFF_INDEX[off]] * iv) * pref
        if rho is not None:
            j = j / rho
        j = j.copy()
        j[geom.pinned] = 0.0
        out.append(j)
    return out[0], out[1]


def line_factor(a, d, jl, ju, dt):
    """Thomas factorisation of M = a + dt d (diagonal), dt jl / dt ju (off
    diagonals) along axis 0, sequential in i and elementwise over the lines:
    inv_i = 1 / (m_i - l_i cp_{i-1}), cp_i = u_i inv_i."""
    n0 = d.shape[0]
    m = a + dt * d
    inv = np.empty_like(d)
    cp = np.empty_like(d)
    for i in range(n0):
        den = m[i] if i == 0 else m[i] - (dt * jl[i]) * cp[i - 1]
        inv[i] = 1.0 / den
        cp[i] = (dt * ju[i]) * inv[i]
    return inv, cp


def line_solve(r, jl, inv, cp, dt):
    """z = M^{-1} r: forward z'_i = (r_i - l_i z'_{i-1}) inv_i, backward
    z_i = z'_i - cp_i z_{i+1}."""
    n0 = r.shape[0]
    z = np.empty_like(r)
    z[0] = r[0] * inv[0]
    for i in range(1, n0):
        z[i] = (r[i] - (dt * jl[i]) * z[i - 1]) * inv[i]
    for i in range(n0 - 2, -1, -1):
        z[i] = z[i] - cp[i] * z[i + 1]
    return z
