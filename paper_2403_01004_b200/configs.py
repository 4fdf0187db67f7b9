"""Seeded synthetic inputs for the BASELINE.json configurations C1-C5.

There is no public dataset for this path: every config is a
recipe.  Builder choices (recorded in DESIGN.md):

* noise "N(0, sigma)" = sigma * sqrt(3) * (u1 + u2 + u3 + u4 - 2), u_t uniform
  from a splitmix64 counter hash of (seed, stream, global cell index, t):
  an Irwin-Hall approximation of a unit normal that any device or host can
  regenerate bit-identically for any sub-block;
* Gaussian bump exp(-(d/w)^2) with d the Euclidean chord distance;
* C3-C5 temperatures in MK (2e4 K -> 0.02), kappa0 = f_c = f_m = rho = 1,
  prefactor (gamma-1) m_p / (2 k) = 1 (m_p = 3, k = 1); counts are invariant
  to the kappa0 scale;
* stretched r grids: C2 geometric ratio 1.01 on [1, 2.5]; C3-C5 geometric on
  [1, 3] with q^(n_r - 1) = 157 (dr_min = 2.56e-4 at n_r = 256);
* C4 step = 1e4 dt_E; C5 step = 5e4 min(dt_E(conduction), dt_E(viscosity)).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import mesh

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
C1_ = np.uint64(0xBF58476D1CE4E5B9)
C2_ = np.uint64(0x94D049BB133111EB)
SQRT3 = math.sqrt(3.0)
TWO_M53 = 2.0 ** -53


def splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * C1_
        z = (z ^ (z >> np.uint64(27))) * C2_
        return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> np.uint64:
    return np.uint64(((seed & 0xFFFFFFFF) << 32 | (stream & 0xFFFF) << 16) & 0xFFFFFFFFFFFFFFFF)


def hash_normal(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Approximately unit-normal noise for global linear indices ``idx``."""
    idx = np.asarray(idx, dtype=np.uint64)
    key = stream_key(seed, stream)
    with np.errstate(over="ignore"):
        base = splitmix64(idx ^ key) * np.uint64(4)
    s = None
    for t in range(4):
        with np.errstate(over="ignore"):
            h = splitmix64(base + np.uint64(t))
        u = (h >> np.uint64(11)).astype(np.float64) * TWO_M53
        s = u if s is None else s + u
    return (s - 2.0) * SQRT3


def block_noise(seed, stream, shape, start=0):
    n = int(np.prod(shape))
    return hash_normal(seed, stream, np.arange(start, start + n, dtype=np.uint64)).reshape(shape)


# ---------------------------------------------------------------- grids

def r_uniform(n, lo, hi):
    return np.linspace(lo, hi, n)


def r_geometric_ratio(n, lo, hi, ratio):
    """r_{i+1} - r_i = dr0 * ratio^i, spanning [lo, hi]."""
    k = np.arange(n - 1)
    d = ratio ** k
    d = d * ((hi - lo) / d.sum())
    r = np.concatenate([[lo], lo + np.cumsum(d)])
    r[-1] = hi
    return r


def r_stretched_c3(n, lo=1.0, hi=3.0, total_ratio=157.0):
    return r_geometric_ratio(n, lo, hi, total_ratio ** (1.0 / (n - 2)))


def spherical_bc(kind="dirichlet"):
    f = mesh.FaceBC(kind)
    return mesh.BoundaryCondition.spherical(f, f)


# ---------------------------------------------------------------- fields

def gaussian_bump(grid, centre=(1.75, math.pi / 2, math.pi), width=0.2):
    R, T, P = grid.meshgrid()
    x, y, z = R * np.sin(T) * np.cos(P), R * np.sin(T) * np.sin(P), R * np.cos(T)
    r0, t0, p0 = centre
    cx, cy, cz = r0 * math.sin(t0) * math.cos(p0), r0 * math.sin(t0) * math.sin(p0), r0 * math.cos(t0)
    d2 = (x - cx) ** 2 + (y - cy) ** 2 + (z - cz) ** 2
    return np.exp(-d2 / (width * width))


def transition_profile(r, T_chromo=0.02, T_corona=1.5, r_tr=1.01, width=0.005):
    return np.array([T_chromo + (T_corona - T_chromo) * 0.5 * (1.0 + math.tanh((x - r_tr) / width)) for x in r])


def temperature(grid, seed, sigma=1e-3, i0=0, n0=None):
    """T = T_prof(r) * (1 + sigma * noise) on axis-0 rows [i0, i0 + n0)."""
    n0 = grid.shape[0] if n0 is None else n0
    prof = transition_profile(grid.coords[0])[i0:i0 + n0]
    shp = (n0, grid.shape[1], grid.shape[2])
    nz = block_noise(seed, 1, shp, start=i0 * grid.shape[1] * grid.shape[2])
    return prof[:, None, None] * (1.0 + sigma * nz)


def dipole_bhat(grid, seed, eps=0.05, i0=0, n0=None):
    """b = normalise(B_dip + eps |B_dip| n), B_dip = (2 cos th / r^3, sin th / r^3, 0)."""
    n0 = grid.shape[0] if n0 is None else n0
    r, th = grid.coords[0][i0:i0 + n0], grid.coords[1]
    ir3 = 1.0 / (r * r * r)
    c2 = np.array([2.0 * math.cos(t) for t in th])
    st = np.array([math.sin(t) for t in th])
    shp = (n0, grid.shape[1], grid.shape[2])
    Br = (c2[None, :] * ir3[:, None])[:, :, None] * np.ones(shp)
    Bt = (st[None, :] * ir3[:, None])[:, :, None] * np.ones(shp)
    mag = np.sqrt(Br * Br + Bt * Bt)
    start = i0 * grid.shape[1] * grid.shape[2]
    a = eps * mag
    bx = Br + a * block_noise(seed, 2, shp, start)
    by = Bt + a * block_noise(seed, 3, shp, start)
    bz = a * block_noise(seed, 4, shp, start)
    nrm = np.sqrt((bx * bx + by * by) + bz * bz)
    return np.stack([bx / nrm, by / nrm, bz / nrm], axis=-1)


def harmonic_tables(grid, seed, n_modes=8, lmax=16):
    """acc[c] = sum_m A_m P_l^m(cos th) cos(m phi + psi) on the (theta, phi) grid, per component."""
    from scipy.special import sph_harm_y

    rng = np.random.default_rng(seed)
    th, ph = grid.coords[1], grid.coords[2]
    out = np.empty((3, grid.shape[1], grid.shape[2]))
    for c in range(3):
        acc = np.zeros((grid.shape[1], grid.shape[2]))
        for _ in range(n_modes):
            l = int(rng.integers(0, lmax + 1))
            m = int(rng.integers(0, l + 1))
            psi = float(rng.uniform(0, 2 * math.pi))
            amp = float(rng.normal())
            Th = np.real(sph_harm_y(l, m, th, 0.0))
            Ph = np.array([math.cos(m * p + psi) for p in ph])
            acc = acc + (amp * Th)[:, None] * Ph[None, :]
        out[c] = acc
    return out


def harmonic_velocity(grid, seed, n_modes=8, lmax=16, checker=0.1, i0=0, n0=None):
    """v_c = sum_m A_m P_l^m(cos th) cos(m phi + psi) + checker (-1)^(i+j+k), per component."""
    n0 = grid.shape[0] if n0 is None else n0
    acc = harmonic_tables(grid, seed, n_modes, lmax)
    shp = (n0, grid.shape[1], grid.shape[2])
    out = np.empty(shp + (3,))
    ii = (np.arange(i0, i0 + n0)[:, None, None] + np.arange(shp[1])[None, :, None] + np.arange(shp[2])[None, None, :])
    cb = np.where(ii % 2 == 0, checker, -checker)
    for c in range(3):
        out[..., c] = acc[c][None, :, :] + cb
    return out


# ---------------------------------------------------------------- device-side generation
# The same recipes evaluated in HBM by the library (pc_gen_*), bit-identical to
# the host functions above: only the 1-D / 2-D tables are built here.

def _dptr(a):
    from . import _lib
    return _lib.dptr(a)


def gen_temperature(field, grid, seed, sigma=1e-3):
    from . import _lib
    prof = np.ascontiguousarray(transition_profile(grid.coords[0]))
    _lib.check(_lib.lib().pc_gen_temperature(field.handle, int(seed), 1, float(sigma), _dptr(prof)), "gen T")
    return field


def gen_dipole(field, grid, seed, eps=0.05):
    from . import _lib
    r, th = grid.coords[0], grid.coords[1]
    ir3 = np.ascontiguousarray(1.0 / (r * r * r))
    c2 = np.array([2.0 * math.cos(t) for t in th])
    st = np.array([math.sin(t) for t in th])
    _lib.check(_lib.lib().pc_gen_dipole(field.handle, int(seed), 2, float(eps), _dptr(ir3), _dptr(c2), _dptr(st)),
               "gen b")
    return field


def gen_harmonic(field, grid, seed, checker=0.1):
    from . import _lib
    acc = np.ascontiguousarray(harmonic_tables(grid, seed))
    _lib.check(_lib.lib().pc_gen_harmonic(field.handle, _dptr(acc), float(checker)), "gen v")
    return field


def gen_radial(field, table):
    from . import _lib
    t = np.ascontiguousarray(np.asarray(table, float))
    _lib.check(_lib.lib().pc_gen_radial(field.handle, _dptr(t)), "gen radial")
    return field


@dataclass
class Workload:
    name: str
    grid: mesh.Grid
    bc: mesh.BoundaryCondition
    ratio: float
    seed: int
    fields: dict = dc_field(default_factory=dict)
    meta: dict = dc_field(default_factory=dict)


def c1(seed=1, n=(48, 48, 96)):
    grid = mesh.build_spherical_grid(r_uniform(n[0], 1.0, 2.5), n[1], n[2])
    bc = spherical_bc("dirichlet")
    u = gaussian_bump(grid) + 0.01 * block_noise(seed, 0, grid.shape)
    u = mesh.apply_dirichlet_values(mesh.Field(grid, u), bc).values[..., 0]
    return Workload("C1", grid, bc, 500.0, seed, {"u": u}, {"tol": 1e-10})


def c2(seed=2, n=(128, 128, 256)):
    grid = mesh.build_spherical_grid(r_geometric_ratio(n[0], 1.0, 2.5, 1.01), n[1], n[2])
    bc = spherical_bc("dirichlet")
    v = harmonic_velocity(grid, seed)
    return Workload("C2", grid, bc, 2000.0, seed, {"v": v}, {"nu": 1.0})


def c3(seed=3, n=(256, 256, 512), host=True):
    """host=False skips the host arrays (the bench generates them in HBM with gen_*)."""
    grid = mesh.build_spherical_grid(r_stretched_c3(n[0]), n[1], n[2])
    bc = spherical_bc("dirichlet")
    fields = {"T": temperature(grid, seed), "b": dipole_bhat(grid, seed)} if host else {}
    return Workload("C3", grid, bc, 1e4, seed, fields, {"m_p": 3.0, "k_B": 1.0})


def c4(seed=4, n=(512, 512, 1024), host=True):
    w = c3(seed, n, host)
    w.name = "C4"
    w.meta["tol"] = 1e-9
    return w


def c5(seed=5, n=(768, 768, 1536), host=False):
    """Coupled conduction (T, b as C3) + viscosity (v as C2) with rho = exp(-10 (r - 1)),
    one MAS step of 5e4 dt_E, dt_E = min over the two operators."""
    grid = mesh.build_spherical_grid(r_stretched_c3(n[0]), n[1], n[2])
    bc = spherical_bc("dirichlet")
    rho_r = np.exp(-10.0 * (grid.coords[0] - 1.0))
    fields = {}
    if host:
        fields = {"T": temperature(grid, seed), "b": dipole_bhat(grid, seed), "v": harmonic_velocity(grid, seed),
                  "rho": rho_r[:, None, None] * np.ones(grid.shape)}
    return Workload("C5", grid, bc, 5e4, seed, fields, {"rho_r": rho_r, "m_p": 3.0, "k_B": 1.0, "nu": 1.0})
