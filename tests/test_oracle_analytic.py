"""Analytic consistency of the spherical operators (the semantics no
reference code pins): the oracle's discrete operators against
closed-form Laplacians, with fitted convergence orders.  The GPU kernels are
bitwise equal to these operators (test_gpu_*), so this pins both.

Grids: r in [1, 2] (n + 1 nodes, Dirichlet ends excluded from the norms),
theta cell-centred (n rows), phi periodic (2n).  Errors are measured in the
rho V-weighted L2 norm (second order everywhere) and the max norm (first
order in the pole rows, where the zero-area pole faces make the theta flux
one-sided)."""
import math

import numpy as np
import pytest

from helpers import oracle_aligned, oracle_scalar
from paper_2403_01004_b200 import configs, mesh

NS = (16, 32, 64)


def _grid(n):
    g = mesh.build_spherical_grid(np.linspace(1.0, 2.0, n + 1), n, 2 * n)
    bc = configs.spherical_bc("dirichlet")
    r, t, p = (np.asarray(c) for c in g.coords)
    R, T, P = np.meshgrid(r, t, p, indexing="ij")
    return g, bc, R, T, P


def _cart(R, T, P):
    return R * np.sin(T) * np.cos(P), R * np.sin(T) * np.sin(P), R * np.cos(T)


def _norms(e, W):
    return float(np.max(np.abs(e))), float(math.sqrt(np.sum(W * e * e) / np.sum(W)))


def _order(errs):
    """Least-squares slope of log(err) against log(h), h = 1/n."""
    h = np.log(1.0 / np.asarray(NS, float))
    return float(np.polyfit(h, np.log(errs), 1)[0])


def _scalar_errors(f, lap):
    out = []
    for n in NS:
        g, bc, R, T, P = _grid(n)
        op = oracle_scalar(g, bc)
        F = op.apply(f(*_cart(R, T, P), R)[None])[0]
        W = op.weights()[0]
        out.append(_norms((F - lap)[1:-1], W[1:-1]))
    return np.array(out)


def test_laplacian_of_r_squared_is_six():
    """The radial flux difference of r^2 is exact: 6 to round-off."""
    e = _scalar_errors(lambda X, Y, Z, R: R * R, 6.0)
    assert np.all(e[:, 0] <= 1e-12 * 6.0 * 100)


@pytest.mark.parametrize("name,f", [
    ("x", lambda X, Y, Z, R: X),
    ("z2-(x2+y2)/2", lambda X, Y, Z, R: Z * Z - 0.5 * (X * X + Y * Y)),
    ("xyz", lambda X, Y, Z, R: X * Y * Z),
])
def test_harmonic_functions_converge_second_order(name, f):
    """Harmonic polynomials: the discrete Laplacian tends to 0 at second
    order in the weighted L2 norm, at least first order in the max norm."""
    e = _scalar_errors(f, 0.0)
    assert np.all(np.diff(e[:, 1]) < 0) and np.all(np.diff(e[:, 0]) < 0)
    assert _order(e[:, 1]) >= 1.8, (name, e)
    assert _order(e[:, 0]) >= 0.9, (name, e)


def _vector(R, T, P, V):
    st, ct, sp, cp = np.sin(T), np.cos(T), np.sin(P), np.cos(P)
    Vx, Vy, Vz = V
    return np.stack([Vx * st * cp + Vy * st * sp + Vz * ct, Vx * ct * cp + Vy * ct * sp - Vz * st,
                     -Vx * sp + Vy * cp])


def test_vector_laplacian_of_constant_field_vanishes():
    """A constant Cartesian vector (z-hat) in spherical components: the
    metric terms cancel exactly, F = 0 to round-off."""
    for n in NS:
        g, bc, R, T, P = _grid(n)
        one = np.ones_like(R)
        op = oracle_scalar(g, bc, ncomp=3, vector_metric=True)
        F = op.apply(_vector(R, T, P, (0 * one, 0 * one, one)))
        assert np.max(np.abs(F[:, 1:-1])) <= 1e-9


def test_vector_laplacian_of_linear_field_converges():
    """(y, z, x) is harmonic per Cartesian component: the vector Laplacian
    with metric terms tends to 0 at second order (weighted L2)."""
    out = []
    for n in NS:
        g, bc, R, T, P = _grid(n)
        X, Y, Z = _cart(R, T, P)
        op = oracle_scalar(g, bc, ncomp=3, vector_metric=True)
        F = op.apply(_vector(R, T, P, (Y, Z, X)))[:, 1:-1]
        W = op.weights()[0][1:-1]
        out.append((float(np.max(np.abs(F))), float(math.sqrt(np.sum(W * F * F) / np.sum(W) / 3))))
    e = np.array(out)
    assert _order(e[:, 1]) >= 1.8, e
    assert _order(e[:, 0]) >= 0.9, e


def test_aligned_radial_field_converges_to_six():
    """Field-aligned conduction with b = r-hat, c = 1 and T = r^2 is the
    radial part of the Laplacian: F -> 6 at second order (both norms)."""
    out = []
    for n in NS:
        g, bc, R, T, P = _grid(n)
        b = np.stack([np.ones_like(R), 0 * R, 0 * R], -1)
        op = oracle_aligned(g, bc, b, np.ones_like(R))
        F = op.apply((R * R)[None])[0]
        W = op.weights()[0]
        out.append(_norms((F - 6.0)[1:-1], W[1:-1]))
    e = np.array(out)
    assert _order(e[:, 1]) >= 1.8, e
    assert _order(e[:, 0]) >= 1.8, e
