"""phi-slab decomposition (BASELINE C4's split) on one GPU.

A phi-slab rank owns the phi columns [k0, k0 + n) of every (r, theta) row
plus one ghost column on each side (pinned, zero inner-product weight),
filled by a periodic NCCL ring.  Two halves are checked here, as for the
r-slabs (test_gpu_slab_local.py, test_gpu_nccl1.py):

* detached ranks (no communicator; ghost columns written from the global
  arrays, exactly what the ring delivers): F, the Gershgorin bound, the
  Jacobi diagonal and the |F| argmax's GLOBAL index of every slab are
  bitwise the single-domain results on its columns;
* one rank with a one-rank NCCL communicator and ghost columns
  (force_ghosts): the ring exchange sends the slab's edge columns to itself,
  so a whole PTL-cycled advance must reproduce the single-rank path (which
  wraps phi in-kernel): RKL2 bitwise, BE+PCG identical iteration counts."""
import numpy as np
import pytest

from helpers import oracle_aligned, oracle_scalar, soa
from oracle import ptl as optl
from paper_2403_01004_b200 import _lib, configs, device, geometry, operators, ptl, schemes

pytestmark = pytest.mark.gpu


def _phi_field(dg, glob_soa):
    """DeviceField holding this rank's phi-slab of a global SoA array + ghost columns."""
    nc, n0, n1, n2 = glob_soa.shape
    k0, n = dg.phi
    f = device.DeviceField(dg, nc)
    f.upload(np.ascontiguousarray(glob_soa[..., k0:k0 + n]), layout=_lib.LAYOUT_SOA)
    ghosts = np.stack([glob_soa[..., (k0 - 1) % n2], glob_soa[..., (k0 + n) % n2]], axis=1)  # (nc, 2, n0, n1)
    f.set_ghost_cols(ghosts)
    return f


def _detached(P, r):
    return device.Context(0, P, r, detached=True, axis=2)


@pytest.mark.parametrize("P", [2, 3, 4])
def test_aligned_phi_slabs_bitwise(gpu_ctx, P):
    w = configs.c5(n=(20, 24, 64), host=True)
    Tg = soa(w.fields["T"][..., None])
    bg = soa(w.fields["b"])
    rg = soa(w.fields["rho"][..., None])
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"], rho=w.fields["rho"])
    Fo = oop.apply(Tg)[0]
    lam, dg_o = oop.bound_and_diag()
    for r in range(P):
        ctx = _detached(P, r)
        try:
            dg = device.device_grid(w.grid, w.bc, ctx)
            k0, n = dg.phi
            assert (k0, n) == geometry.slab_bounds(64, P, r) and dg.shape == (20, 24, n + 2)
            T, b, rho = _phi_field(dg, Tg), _phi_field(dg, bg), _phi_field(dg, rg)
            op = operators.DiffusionOperator.aligned(
                operators.AlignedConductionConfig(b_hat=b, rho=rho, m_p=3.0, k_B=1.0, bc=w.bc))
            op.freeze(T)
            dop = op.device_op(w.grid, 1, ctx)
            F = device.DeviceField(dg, 1)
            dop.apply(T, F)
            assert np.array_equal(F.download()[..., 0], Fo[..., k0:k0 + n]), f"rank {r}/{P}: F differs"
            loc = float(np.max(lam[0][..., k0:k0 + n]))
            assert dop.dt_euler == 2.0 / loc, f"rank {r}/{P}: bound differs"
            d = dop.diagonal().download()[..., 0]
            assert np.array_equal(d, dg_o[0][..., k0:k0 + n]), f"rank {r}/{P}: Jacobi diagonal differs"
            del T, b, rho, op, dop, F
        finally:
            ctx.close()


@pytest.mark.parametrize("P", [2, 4])
def test_viscous_phi_slabs_bitwise(gpu_ctx, P):
    w = configs.c5(n=(16, 12, 32), host=True)
    vg = soa(w.fields["v"])
    rg = soa(w.fields["rho"][..., None])
    oop = oracle_scalar(w.grid, w.bc, nu=1.0, rho=w.fields["rho"], ncomp=3, vector_metric=True)
    Fo = oop.apply(vg)
    for r in range(P):
        ctx = _detached(P, r)
        try:
            dg = device.device_grid(w.grid, w.bc, ctx)
            k0, n = dg.phi
            v, rho = _phi_field(dg, vg), _phi_field(dg, rg)
            op = operators.DiffusionOperator.scalar(
                operators.ScalarDiffusionConfig(nu=1.0, rho=rho, bc=w.bc, vector_metric=True), 3)
            dop = op.device_op(w.grid, 3, ctx)
            F = device.DeviceField(dg, 3)
            dop.apply(v, F)
            assert np.array_equal(soa(F.download()), Fo[..., k0:k0 + n]), f"rank {r}/{P}: F differs"
            del v, rho, op, dop, F
        finally:
            ctx.close()


def test_phi_slab_argmax_index_is_global(gpu_ctx):
    from ctypes import byref, c_double, c_int, c_int64
    w = configs.c3(n=(16, 20, 64))
    Tg = soa(w.fields["T"][..., None])
    bg = soa(w.fields["b"])
    Fo = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"]).apply(Tg)[0]
    P = 4
    best = []
    for r in range(P):
        ctx = _detached(P, r)
        try:
            dg = device.device_grid(w.grid, w.bc, ctx)
            k0, n = dg.phi
            T, b = _phi_field(dg, Tg), _phi_field(dg, bg)
            op = operators.DiffusionOperator.aligned(
                operators.AlignedConductionConfig(b_hat=b, m_p=3.0, k_B=1.0, bc=w.bc))
            op.freeze(T)
            dop = op.device_op(w.grid, 1, ctx)
            F = device.DeviceField(dg, 1)
            dop.apply(T, F)
            F.set_ghost_cols(np.stack([Fo[None, ..., (k0 - 1) % 64], Fo[None, ..., (k0 + n) % 64]], axis=1))
            v, lim, k = c_double(), c_int(), c_int64()
            _lib.check(_lib.lib().pc_ptl(dg.handle, T.handle, F.handle, 1e-12, 0, byref(v), byref(lim), byref(k)),
                       "pc_ptl")
            blk = np.abs(Fo[..., k0:k0 + n])
            li = np.unravel_index(int(np.argmax(blk)), blk.shape)
            assert k.value == (li[0] * Fo.shape[1] + li[1]) * Fo.shape[2] + li[2] + k0, f"rank {r}: not global"
            best.append((float(blk[li]), k.value))
            del T, b, op, dop, F
        finally:
            ctx.close()
    gi = int(np.argmax(np.abs(Fo)))
    assert min(best, key=lambda t: (-t[0], t[1]))[1] == gi


@pytest.fixture(scope="module")
def nccl_phi_ctx():
    mp = pytest.MonkeyPatch()
    mp.setenv("PC_FORCE_NCCL", "1")
    ctx = device.Context(0, axis=2)
    mp.undo()
    yield ctx
    ctx.close()


def _self_ring_grid(ctx, grid, bc):
    dg = device.DeviceGrid(grid, bc, ctx, force_ghosts=True)
    assert dg.phi == (0, grid.shape[2])
    ctx._grids[(id(grid), id(bc))] = (grid, bc, dg)
    return dg


@pytest.mark.parametrize("kind", ["rkl2", "backward_euler"])
def test_phi_ring_self_exchange_cycle(gpu_ctx, nccl_phi_ctx, kind):
    """A whole PTL-cycled C3-recipe advance on a one-rank phi ring (ghost
    columns from ncclSend/ncclRecv to itself every stage / PCG iteration, the
    F ghost columns for the PTL pairs) == the single-rank in-kernel wrap."""
    w = configs.c3(n=(20, 24, 64))
    T = operators.Field(w.grid, w.fields["T"])
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
    _self_ring_grid(nccl_phi_ctx, w.grid, w.bc)
    res = []
    for ctx in (gpu_ctx, nccl_phi_ctx):
        op = operators.DiffusionOperator.aligned(cfg, T)
        dtE = op.device_op(w.grid, 1, ctx).dt_euler
        out, rep = ptl.cycle_operator(op, schemes.SchemeConfig(kind, tol=1e-9), T, 1e3 * dtE, ctx=ctx)
        res.append((dtE, [e.iters for e in rep.entries], out.values.copy()))
    assert res[0][0] == res[1][0]
    assert res[0][1] == res[1][1]
    if kind == "rkl2":
        assert np.array_equal(res[0][2], res[1][2])
    else:
        assert np.linalg.norm(res[0][2] - res[1][2]) <= 1e-10 * np.linalg.norm(res[0][2])
    # and both are the oracle's
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme(kind, tol=1e-9), soa(w.fields["T"][..., None]),
                                   1e3 * res[0][0], dt_euler=res[0][0])
    assert res[1][1] == [r.iters for r in repo]


def test_phi_ring_viscous_and_audit(gpu_ctx, nccl_phi_ctx):
    """Vector viscosity with rho on the one-rank phi ring, PTL audit mode
    (every pair, each counted once across the ring): bitwise the single rank."""
    w = configs.c5(n=(16, 12, 32), host=True)
    v = operators.Field(w.grid, w.fields["v"])
    rho = w.fields["rho"][..., None]
    _self_ring_grid(nccl_phi_ctx, w.grid, w.bc)
    res = []
    for ctx in (gpu_ctx, nccl_phi_ctx):
        op = operators.DiffusionOperator.scalar(
            operators.ScalarDiffusionConfig(nu=1.0, rho=operators.Field(w.grid, rho), bc=w.bc, vector_metric=True), 3)
        dtE = op.device_op(w.grid, 3, ctx).dt_euler
        out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), v, 300 * dtE,
                                      ptl.PtlConfig(check_all_points=True), ctx=ctx)
        res.append((dtE, [(e.dt, e.iters) for e in rep.entries], out.values.copy()))
    assert res[0][0] == res[1][0]
    assert res[0][1] == res[1][1]
    assert np.array_equal(res[0][2], res[1][2])
