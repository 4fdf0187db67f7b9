"""The r-slab kernels on one GPU.

Only one GPU is available to this build, so the NCCL exchange itself cannot
run here; what can run is everything a rank does locally.  Each rank of an
r-slab decomposition is built on its own *detached* context (the library's
test hook: no communicator, collectives skipped) and its axis-0 ghost planes
are filled from the global arrays, exactly what the halo exchange delivers.
Every slab's F (and Gershgorin bound) must then be bitwise the single-domain
result restricted to the slab: this checks the slab geometry tables, the
ghost-plane reads of the marching kernels (TMA and cp.async staging), the
beta-on-ghost-planes freeze and the coefficient ghost planes of the viscous
operator.  (The exchange and reductions are covered by the gloo restatement,
tests/test_multirank_gloo.py.)"""
import numpy as np
import pytest

from helpers import oracle_aligned, oracle_geometry, oracle_scalar, soa
from paper_2403_01004_b200 import _lib, configs, device, geometry, operators

pytestmark = pytest.mark.gpu


def _slab_field(dg, glob_soa):
    """DeviceField holding this rank's slab of a global SoA array (+ ghosts)."""
    nc = glob_soa.shape[0]
    n0 = glob_soa.shape[1]
    f = device.DeviceField(dg, nc)
    i0, n = dg.i0, dg.n0_local
    f.upload(np.ascontiguousarray(glob_soa[:, i0:i0 + n]), layout=_lib.LAYOUT_SOA)
    if dg.ghost_lo:
        f.set_ghost(0, glob_soa[:, (i0 - 1) % n0])
    if dg.ghost_hi:
        f.set_ghost(1, glob_soa[:, (i0 + n) % n0])
    return f


@pytest.mark.parametrize("n", [(36, 20, 64), (30, 24, 48)], ids=["tma", "cpasync"])
@pytest.mark.parametrize("P", [2, 3])
def test_aligned_slabs_bitwise(gpu_ctx, n, P):
    w = configs.c5(n=n, host=True)
    Tg = soa(w.fields["T"][..., None])
    bg = soa(w.fields["b"])
    rg = soa(w.fields["rho"][..., None])
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"], rho=w.fields["rho"])
    Fo = oop.apply(Tg)[0]
    lam, dg_o = oop.bound_and_diag()
    for r in range(P):
        ctx = device.Context(0, P, r, detached=True)
        try:
            dg = device.device_grid(w.grid, w.bc, ctx)
            assert (dg.i0, dg.n0_local) == geometry.slab_bounds(n[0], P, r)
            T = _slab_field(dg, Tg)
            b = _slab_field(dg, bg)
            rho = _slab_field(dg, rg)
            cfg = operators.AlignedConductionConfig(b_hat=b, rho=rho, m_p=3.0, k_B=1.0, bc=w.bc)
            op = operators.DiffusionOperator.aligned(cfg)
            op.freeze(T)
            dop = op.device_op(w.grid, 1, ctx)
            F = device.DeviceField(dg, 1)
            dop.apply(T, F)
            i0, nl = dg.i0, dg.n0_local
            assert np.array_equal(F.download_planes(0, nl)[0], Fo[i0:i0 + nl]), f"rank {r}/{P}: F differs"
            # local Gershgorin bound (detached: no allreduce) = max over the slab's rows
            loc = float(np.max(lam[0][i0:i0 + nl]))
            assert dop.dt_euler == (2.0 / loc if loc > 0 else float("inf")), f"rank {r}/{P}: bound differs"
            d = dop.diagonal().download_planes(0, nl)[0]
            assert np.array_equal(d, dg_o[0][i0:i0 + nl]), f"rank {r}/{P}: Jacobi diagonal differs"
            del T, b, rho, op, dop, F
        finally:
            ctx.close()


@pytest.mark.parametrize("P", [2, 4])
def test_viscous_rho_slabs_bitwise(gpu_ctx, P):
    """C5 viscosity: D = nu rho is read at the axis-0 neighbours, so the rho
    ghost planes matter (refreshed by the operator's freeze)."""
    w = configs.c5(n=(16, 12, 32), host=True)
    vg = soa(w.fields["v"])
    rg = soa(w.fields["rho"][..., None])
    oop = oracle_scalar(w.grid, w.bc, nu=1.0, rho=w.fields["rho"], ncomp=3, vector_metric=True)
    Fo = oop.apply(vg)
    for r in range(P):
        ctx = device.Context(0, P, r, detached=True)
        try:
            dg = device.device_grid(w.grid, w.bc, ctx)
            v = _slab_field(dg, vg)
            rho = _slab_field(dg, rg)
            rho_g = rho  # the operator must not rely on host copies
            cfg = operators.ScalarDiffusionConfig(nu=1.0, rho=rho_g, bc=w.bc, vector_metric=True)
            op = operators.DiffusionOperator.scalar(cfg, 3)
            dop = op.device_op(w.grid, 3, ctx)
            F = device.DeviceField(dg, 3)
            dop.apply(v, F)
            i0, nl = dg.i0, dg.n0_local
            assert np.array_equal(F.download_planes(0, nl), Fo[:, i0:i0 + nl]), f"rank {r}/{P}: F differs"
            del v, rho, rho_g, op, dop, F
        finally:
            ctx.close()


def test_argmax_index_is_global_on_slabs(gpu_ctx):
    """The |F| argmax a rank reports (before the allgather) carries the GLOBAL
    AoS index of its slab's maximum."""
    from ctypes import byref, c_double, c_int, c_int64
    w = configs.c3(n=(24, 20, 64))
    Tg = soa(w.fields["T"][..., None])
    bg = soa(w.fields["b"])
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
    Fo = oop.apply(Tg)[0]
    P = 3
    for r in range(P):
        ctx = device.Context(0, P, r, detached=True)
        try:
            dg = device.device_grid(w.grid, w.bc, ctx)
            T = _slab_field(dg, Tg)
            b = _slab_field(dg, bg)
            op = operators.DiffusionOperator.aligned(
                operators.AlignedConductionConfig(b_hat=b, m_p=3.0, k_B=1.0, bc=w.bc))
            op.freeze(T)
            dop = op.device_op(w.grid, 1, ctx)
            F = device.DeviceField(dg, 1)
            dop.apply(T, F)
            i0, nl = dg.i0, dg.n0_local
            F.set_ghost(0, np.zeros((1,) + Fo.shape[1:]))
            F.set_ghost(1, np.zeros((1,) + Fo.shape[1:]))
            v, lim, k = c_double(), c_int(), c_int64()
            _lib.check(_lib.lib().pc_ptl(dg.handle, T.handle, F.handle, 1e-12, 0, byref(v), byref(lim), byref(k)),
                       "pc_ptl")
            blk = np.abs(Fo[i0:i0 + nl])
            loc = int(np.argmax(blk))
            assert k.value == loc + i0 * Fo.shape[1] * Fo.shape[2], f"rank {r}: argmax index not global"
            del T, b, op, dop, F
        finally:
            ctx.close()


def test_ptl_pairs_across_slab_boundaries(gpu_ctx):
    """Each rank's PTL pairs at its |F| maximum, planted on the slab's FIRST
    (then LAST) plane so that one pair reaches into the ghost plane, equal the
    pairs of the global arrays at that node (bitwise)."""
    from ctypes import byref, c_double, c_int, c_int64
    from oracle.ptl import neighbours
    w = configs.c3(n=(24, 20, 64))
    geom = oracle_geometry(w.grid, w.bc)
    rng = np.random.default_rng(7)
    P = 3
    for side in (0, 1):
        u = rng.normal(size=(1,) + geom.shape)
        F = rng.normal(size=(1,) + geom.shape)
        for r in range(P):
            i0, nl = geometry.slab_bounds(geom.shape[0], P, r)
            pi = i0 if side == 0 else i0 + nl - 1
            F[0, pi, 7, 11] = 50.0 + r  # this slab's maximum
            u[0, pi, 7, 11] = 3.0       # du of one sign against every neighbour ...
            F[0, pi, 7, 11] *= -1.0     # ... dF of the other: every pair is a candidate
        for r in range(P):
            ctx = device.Context(0, P, r, detached=True)
            try:
                dg = device.device_grid(w.grid, w.bc, ctx)
                uf, Ff = _slab_field(dg, u), _slab_field(dg, F)
                v, lim, k = c_double(), c_int(), c_int64()
                _lib.check(_lib.lib().pc_ptl(dg.handle, uf.handle, Ff.handle, 1e-12, 0, byref(v), byref(lim),
                                             byref(k)), "pc_ptl")
                i0, nl = dg.i0, dg.n0_local
                pt = (i0 if side == 0 else i0 + nl - 1, 7, 11)
                thr = 1e-12 * abs(F[(0,) + pt])
                best = None
                for nb in neighbours(geom, pt):
                    du = u[(0,) + pt] - u[(0,) + nb]
                    dF = F[(0,) + pt] - F[(0,) + nb]
                    if du != 0.0 and abs(dF) > thr and du * dF < 0.0:
                        best = -du / dF if best is None else min(best, -du / dF)
                assert k.value == (pt[0] * geom.shape[1] + pt[1]) * geom.shape[2] + pt[2]
                assert lim.value == 1 and v.value == best, f"rank {r}: PTL pairs differ"
                del uf, Ff
            finally:
                ctx.close()
