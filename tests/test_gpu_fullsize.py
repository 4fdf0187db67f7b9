"""Full-size parity (BASELINE.json configs C3 and C5 at their own grid sizes).

The oracle cannot evaluate a 33.5 M / 906 M cell grid in seconds, so the GPU
runs the FULL grid and the oracle checks it on axis-0 windows: every stencil
has radius 1, so F on planes [a, b) depends only on planes [a-1, b+1), and s
STS stages only on [a-s, b+s) (helpers.window_geometry).  Inputs are the
seeded recipes, generated in HBM by the library and on the host for the window
only (configs.temperature / dipole_bhat / harmonic_velocity take i0, n0).
Size-independent properties (determinism, exact linearity under a power-of-two
scaling, constants in the kernel) cover the whole grid.  Bar: bitwise.
"""
import gc

import numpy as np
import pytest

from helpers import oracle_geometry, soa, window_geometry
from oracle import operators as oops
from oracle import ptl as optl
from oracle import schemes as osch
from paper_2403_01004_b200 import _lib, configs, device, operators

pytestmark = pytest.mark.gpu


def _conduction(w, ctx, rho=False):
    dg = device.device_grid(w.grid, w.bc, ctx)
    b = configs.gen_dipole(device.DeviceField(dg, 3), w.grid, w.seed)
    T = configs.gen_temperature(device.DeviceField(dg, 1), w.grid, w.seed)
    r = configs.gen_radial(device.DeviceField(dg, 1), w.meta["rho_r"]) if rho else None
    cfg = operators.AlignedConductionConfig(b_hat=b, rho=r, m_p=3.0, k_B=1.0, bc=w.bc)
    op = operators.DiffusionOperator.aligned(cfg)
    op.freeze(T)
    return dg, T, op, op.device_op(w.grid, 1, ctx)


def _oracle_conduction(w, a, b, rho=False):
    gw = window_geometry(oracle_geometry(w.grid, w.bc), a, b)
    T = configs.temperature(w.grid, w.seed, i0=a, n0=b - a)
    bh = configs.dipole_bhat(w.grid, w.seed, i0=a, n0=b - a)
    c = oops.aligned_coefficient(T, 1.0, None, 1e-10)
    r3 = w.meta["rho_r"][a:b, None, None] * np.ones(T.shape) if rho else None
    return optl.OracleOperator(gw, "aligned", 1, None, r3, False, soa(bh), c, 1.0), T[None]


def _windows(n0, width=3):
    """First planes, a window starting at n0/2 (an r-chunk start of the marching
    kernels: the prologue/first-refill hand-off), last planes."""
    mid = n0 // 2
    return [(0, width), (mid, mid + width), (n0 - width, n0)]


def _check_apply_windows(w, dg, T, dop, rho=False):
    F = device.DeviceField(dg, 1)
    dop.apply(T, F)
    n0 = dg.shape[0]
    for a, b in _windows(n0):
        lo, hi = max(a - 1, 0), min(b + 1, n0)
        oop, To = _oracle_conduction(w, lo, hi, rho)
        Fo = oop.apply(To)[0][a - lo:b - lo]
        Fg = F.download_planes(a, b - a)[0]
        assert np.array_equal(Fg, Fo), f"F differs from the oracle on planes [{a}, {b})"
    return F


def _check_sts_windows(w, dg, T, dop, s, rho=False):
    """s fixed RKL2 stages at dt = 0.9 dt_E (s^2 + s - 2) / 4 (inside the stability interval)."""
    dtE = dop.dt_euler
    dt = 0.9 * dtE * (s * s + s - 2) / 4.0
    u = T.clone()
    _lib.check(_lib.lib().pc_step_sts(dop.handle, u.handle, float(dt), _lib.RKL2, int(s), None), "step_sts")
    n0 = dg.shape[0]
    for a, b in _windows(n0, 2):
        lo, hi = max(a - s - 1, 0), min(b + s + 1, n0)
        oop, To = _oracle_conduction(w, lo, hi, rho)
        uo = osch.sts_step(oop.apply, To, oop.apply(To), dt, s, "rkl2", oop.geom.pinned)
        ug = u.download_planes(a, b - a)[0]
        assert np.array_equal(ug, uo[0][a - lo:b - lo]), f"stage {s} field differs on planes [{a}, {b})"


@pytest.fixture(scope="module")
def c3full(gpu_ctx):
    w = configs.c3(host=False)
    dg, T, op, dop = _conduction(w, gpu_ctx)
    yield w, dg, T, op, dop
    del T, op, dop
    gc.collect()


def test_c3_full_apply_windows_bitwise(c3full):
    w, dg, T, op, dop = c3full
    _check_apply_windows(w, dg, T, dop)


def test_c3_full_rkl2_stages_windows_bitwise(c3full):
    w, dg, T, op, dop = c3full
    _check_sts_windows(w, dg, T, dop, 6)


def test_c3_full_properties(c3full):
    """Whole-grid properties of the fused kernel: deterministic, exactly
    linear under x2 (no rounding in a power-of-two scaling), zero on a constant."""
    w, dg, T, op, dop = c3full
    F1, F2, F3 = (device.DeviceField(dg, 1) for _ in range(3))
    dop.apply(T, F1)
    dop.apply(T, F2)
    a1 = F1.download_planes(0, dg.shape[0])
    assert np.array_equal(a1, F2.download_planes(0, dg.shape[0])), "two evaluations differ"
    T2 = device.DeviceField(dg, 1)
    T2.upload(2.0 * T.download_planes(0, dg.shape[0]), _lib.LAYOUT_SOA)
    dop.apply(T2, F3)
    assert np.array_equal(F3.download_planes(0, dg.shape[0]), 2.0 * a1), "F(2T) != 2 F(T)"
    T2.fill(0.75)
    dop.apply(T2, F3)
    assert not np.any(F3.download_planes(0, dg.shape[0])), "F(const) != 0"
    assert np.isfinite(dop.dt_euler) and dop.dt_euler > 0.0


@pytest.fixture(scope="module")
def c5cond(gpu_ctx):
    w = configs.c5()
    dg, T, op, dop = _conduction(w, gpu_ctx, rho=True)
    yield w, dg, T, op, dop
    del T, op, dop
    gc.collect()


def test_c5_full_conduction_windows_bitwise(c5cond):
    """C5 768x768x1536, rho field (the RHO instantiation of the TMA march)."""
    w, dg, T, op, dop = c5cond
    F = _check_apply_windows(w, dg, T, dop, rho=True)
    del F
    _check_sts_windows(w, dg, T, dop, 4, rho=True)


def test_c5_full_viscosity_windows_bitwise(gpu_ctx):
    w = configs.c5()
    dg = device.device_grid(w.grid, w.bc, gpu_ctx)
    rho = configs.gen_radial(device.DeviceField(dg, 1), w.meta["rho_r"])
    v = configs.gen_harmonic(device.DeviceField(dg, 3), w.grid, w.seed)
    cfg = operators.ScalarDiffusionConfig(nu=1.0, rho=rho, bc=w.bc, vector_metric=True)
    op = operators.DiffusionOperator.scalar(cfg, 3)
    dop = op.device_op(w.grid, 3, gpu_ctx)
    F, F2 = device.DeviceField(dg, 3), device.DeviceField(dg, 3)
    dop.apply(v, F)
    dop.apply(v, F2)
    geom = oracle_geometry(w.grid, w.bc)
    n0 = dg.shape[0]
    for a, b in _windows(n0):
        lo, hi = max(a - 1, 0), min(b + 1, n0)
        gw = window_geometry(geom, lo, hi)
        r3 = w.meta["rho_r"][lo:hi, None, None] * np.ones((hi - lo,) + tuple(dg.shape[1:]))
        oop = optl.OracleOperator(gw, "scalar", 3, np.full(r3.shape, 1.0) * r3, r3, True)
        vo = soa(configs.harmonic_velocity(w.grid, w.seed, i0=lo, n0=hi - lo))
        Fo = oop.apply(vo)[:, a - lo:b - lo]
        Fg = F.download_planes(a, b - a)
        assert np.array_equal(Fg, F2.download_planes(a, b - a)), f"two evaluations differ on planes [{a}, {b})"
        bad = np.argwhere(Fg != Fo)
        assert bad.size == 0, (f"viscous F differs on planes [{a}, {b}): {len(bad)} nodes, first {bad[:3].tolist()}, "
                               f"max |diff| {np.max(np.abs(Fg - Fo)):.3e}, max |F| {np.max(np.abs(Fo)):.3e}")
    del F, F2, v, rho, op, dop
    gc.collect()
