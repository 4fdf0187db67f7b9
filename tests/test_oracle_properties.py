"""Property invariants of the SPEC checked on the
CPU oracle over random small grids (hypothesis).  The GPU path is bitwise
equal to the oracle (test_gpu_*), so these properties hold for it too.

* rho V-symmetry of every operator: (u, F(v))_W == (v, F(u))_W;
* negative semi-definiteness: (u, F(u))_W <= 0;
* conservation with no pinned nodes: sum W F(u) == 0 (up to rounding);
* a constant field is a null vector: F(const) == 0 exactly.
Spherical and Cartesian metrics, scalar (with rho), vector viscosity and the
field-aligned operator."""
import numpy as np
from hypothesis import given, settings, strategies as st

from helpers import oracle_aligned, oracle_scalar, soa
from paper_2403_01004_b200 import configs, mesh


def _sph_grid(n0, n1, n2, seed):
    rng = np.random.default_rng(seed)
    r = 1.0 + np.cumsum(np.concatenate([[0.0], rng.uniform(0.05, 0.2, n0 - 1)]))
    return mesh.build_spherical_grid(r, n1, n2)


def _cart_grid(n0, n1, n2, seed):
    rng = np.random.default_rng(seed)
    cs = [np.cumsum(np.concatenate([[0.0], rng.uniform(0.5, 1.5, n - 1)])) for n in (n0, n1, n2)]
    return mesh.build_grid([n0, n1, n2], coords=cs)


def _ops(kind, metric, n, seed):
    """(oracle operator, ncomp) on a grid with no pinned node."""
    rng = np.random.default_rng(seed + 17)
    if metric == "spherical":
        g = _sph_grid(*n, seed)
        bc = mesh.BoundaryCondition.spherical(mesh.FaceBC("neumann"), mesh.FaceBC("neumann"))
    else:
        g = _cart_grid(*n, seed)
        bc = mesh.BoundaryCondition(((mesh.FaceBC("neumann"), mesh.FaceBC("neumann")),
                                     (mesh.FaceBC("periodic"), mesh.FaceBC("periodic")),
                                     (mesh.FaceBC("neumann"), mesh.FaceBC("neumann"))))
    rho = rng.uniform(0.5, 2.0, g.shape)
    if kind == "scalar":
        return oracle_scalar(g, bc, nu=1.0, rho=rho), 1
    if kind == "vector":
        return oracle_scalar(g, bc, nu=1.0, rho=rho, ncomp=3, vector_metric=(metric == "spherical")), 3
    b = rng.normal(size=g.shape + (3,))
    b /= np.linalg.norm(b, axis=-1, keepdims=True)
    T0 = rng.uniform(0.5, 2.0, g.shape)
    return oracle_aligned(g, bc, b, T0, rho=rho), 1


dims = st.tuples(st.integers(3, 6), st.integers(3, 6), st.integers(3, 7))
kinds = st.sampled_from(["scalar", "vector", "aligned"])
metrics = st.sampled_from(["spherical", "cartesian"])


@settings(max_examples=30, deadline=None)
@given(kind=kinds, metric=metrics, n=dims, seed=st.integers(0, 10**6))
def test_weighted_symmetry_and_definiteness(kind, metric, n, seed):
    op, nc = _ops(kind, metric, n, seed)
    assert not op.geom.pinned.any()
    rng = np.random.default_rng(seed)
    u = rng.normal(size=(nc,) + op.geom.shape)
    v = rng.normal(size=(nc,) + op.geom.shape)
    W = op.weights()
    Fu, Fv = op.apply(u), op.apply(v)
    a, b = np.sum(W * u * Fv), np.sum(W * v * Fu)
    scale = np.sum(np.abs(W * u * Fv)) + np.sum(np.abs(W * v * Fu))
    assert abs(a - b) <= 1e-12 * scale
    q = np.sum(W * u * Fu)
    assert q <= 1e-12 * np.sum(np.abs(W * u * Fu))


@settings(max_examples=30, deadline=None)
@given(kind=kinds, metric=metrics, n=dims, seed=st.integers(0, 10**6))
def test_conservation_and_constant_null_vector(kind, metric, n, seed):
    op, nc = _ops(kind, metric, n, seed)
    rng = np.random.default_rng(seed)
    u = rng.normal(size=(nc,) + op.geom.shape)
    W = op.weights()
    Fu = op.apply(u)
    if kind != "vector" or metric == "cartesian":  # the vector metric rotates components: sum per component not conserved
        assert abs(np.sum(W * Fu)) <= 1e-12 * np.sum(np.abs(W * Fu))
    c = np.full((nc,) + op.geom.shape, 1.7)
    if kind == "vector" and metric == "spherical":
        return  # a constant (v_r, v_theta, v_phi) is not a constant Cartesian vector
    assert not np.any(op.apply(c))


def test_c3_recipe_operator_is_dissipative():
    """The C3 recipe (Dirichlet r ends, axis, periodic phi) at a reduced size:
    on the free nodes the aligned operator is W-symmetric and dissipative."""
    w = configs.c3(n=(10, 8, 16))
    op = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
    free = ~op.geom.pinned
    rng = np.random.default_rng(3)
    u = rng.normal(size=(1,) + op.geom.shape) * free
    v = rng.normal(size=(1,) + op.geom.shape) * free
    W = op.weights()
    a = np.sum((W * u * op.apply(v))[:, free])
    b = np.sum((W * v * op.apply(u))[:, free])
    assert abs(a - b) <= 1e-12 * (abs(a) + abs(b))
    assert np.sum((W * u * op.apply(u))[:, free]) < 0.0
    assert np.array_equal(soa(w.fields["T"][..., None]).shape, (1,) + op.geom.shape)
