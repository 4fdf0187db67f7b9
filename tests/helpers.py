"""Test-side adapters between the product API and the CPU oracle."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle.geometry import build_geometry  # noqa: E402
from oracle import ptl as optl  # noqa: E402


def oracle_geometry(grid, bc):
    kinds = [(lo.kind, hi.kind) for lo, hi in bc.faces]
    return build_geometry(list(grid.coords), kinds, getattr(grid, "metric", "cartesian"))


def soa(values, ncomp=None):
    """(grid..., ncomp) AoS -> (ncomp, n0, n1, n2) SoA padded to 3 axes."""
    v = np.asarray(values, float)
    if ncomp is None:
        ncomp = v.shape[-1] if v.ndim >= 2 and v.shape[-1] in (1, 3) and v.ndim in (2, 3, 4) else 1
    v = np.moveaxis(v, -1, 0)
    while v.ndim < 4:
        v = v[..., None]
    return np.ascontiguousarray(v)


def aos(u_soa, dims):
    v = np.moveaxis(u_soa, 0, -1)
    return v.reshape(v.shape[:dims] + v.shape[3:]) if dims < 3 else v


def oracle_scalar(grid, bc, nu=1.0, rho=None, ncomp=1, vector_metric=False):
    g = oracle_geometry(grid, bc)
    D = None
    if isinstance(nu, float) and (rho is None or isinstance(rho, float)):
        D = nu if rho is None else nu * rho
        rho3 = None if rho is None else np.full(g.shape, rho)
    else:
        nu3 = np.broadcast_to(nu, g.shape) if isinstance(nu, float) else np.asarray(nu, float).reshape(g.shape)
        r3 = None if rho is None else (np.full(g.shape, rho) if isinstance(rho, float) else np.asarray(rho, float).reshape(g.shape))
        D = nu3 if r3 is None else np.full(g.shape, nu) * r3 if isinstance(nu, float) else nu3 * r3
        rho3 = r3
    return optl.OracleOperator(g, "scalar", ncomp, D, rho3, vector_metric and grid.metric == "spherical" and ncomp == 3)


def oracle_aligned(grid, bc, b_aos, T0, pref=1.0, rho=None, kappa0=1.0, T_floor=1e-10):
    from oracle import operators as oops
    g = oracle_geometry(grid, bc)
    b = soa(b_aos)
    c = oops.aligned_coefficient(np.asarray(T0, float).reshape(g.shape), kappa0, None, T_floor)
    r3 = None if rho is None else np.asarray(rho, float).reshape(g.shape)
    return optl.OracleOperator(g, "aligned", 1, None, r3, False, b, c, pref)


def window_geometry(geom, a, b):
    """The oracle geometry restricted to axis-0 planes [a, b) of a global
    geometry (2-D tables sliced, pinned rows kept, axis 0 not periodic): an
    operator evaluated on it is exact on every plane whose axis-0 neighbours
    lie inside the window, so windows of a full-size grid check the GPU at
    full size (oracle/distributed.py Slab slicing)."""
    from oracle.distributed import Slab
    s = Slab.__new__(Slab)
    s.i0, s.n, s.glo, s.ghi = a, b - a, 0, 0
    return s._slice_geometry(geom)
