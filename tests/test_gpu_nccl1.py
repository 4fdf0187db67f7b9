"""The multi-rank collectives through NCCL on ONE GPU: a context with a
one-rank communicator (PC_FORCE_NCCL test hook) sends every reduction of the
r-slab path through NCCL -- Gershgorin allreduce(max), the allgathered |F|
argmax and its combine kernel, the PTL allreduce(min) (and the audit mode's
u64 min), the split PCG reductions finished by k_pcg_fin, the overlapped
stage launches on the communication stream -- and must reproduce the oracle
exactly as the plain single-rank path does."""
import numpy as np
import pytest

from helpers import oracle_aligned, oracle_scalar, soa
from oracle import ptl as optl
from paper_2403_01004_b200 import configs, device, operators, ptl, schemes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_ctx():
    mp = pytest.MonkeyPatch()
    mp.setenv("PC_FORCE_NCCL", "1")
    ctx = device.Context(0)
    mp.undo()
    yield ctx
    ctx.close()


@pytest.mark.parametrize("kind,check_all", [("rkl2", False), ("backward_euler", False), ("rkl2", True)])
def test_aligned_through_nccl(gpu_ctx, nccl_ctx, kind, check_all):
    w = configs.c3(n=(24, 40, 64))
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
    T = operators.Field(w.grid, w.fields["T"])
    op = operators.DiffusionOperator.aligned(cfg, T)
    dtE = op.device_op(w.grid, 1, nccl_ctx).dt_euler
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
    assert dtE == oop.euler_dt()
    sc = schemes.SchemeConfig(kind, tol=1e-9)
    ratio = 300.0 if check_all else 1e4  # the audit mode cycles far more often (oracle cost)
    out, rep = ptl.cycle_operator(op, sc, T, ratio * dtE, ptl.PtlConfig(check_all_points=check_all), ctx=nccl_ctx)
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme(kind, tol=1e-9), soa(w.fields["T"][..., None]),
                                   ratio * dtE, dt_euler=dtE, check_all=check_all)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    a, b = out.values[..., 0], uo[0]
    if kind == "rkl2":
        assert np.array_equal(a, b)
    else:
        assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)


def test_viscous_through_nccl(gpu_ctx, nccl_ctx):
    w = configs.c2(n=(40, 24, 64))
    cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc, vector_metric=True)
    op = operators.DiffusionOperator.scalar(cfg, 3)
    v = operators.Field(w.grid, w.fields["v"])
    dtE = op.device_op(w.grid, 3, nccl_ctx).dt_euler
    oop = oracle_scalar(w.grid, w.bc, ncomp=3, vector_metric=True)
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), v, 200 * dtE, ctx=nccl_ctx)
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(w.fields["v"]), 200 * dtE, dt_euler=dtE)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    assert np.array_equal(np.moveaxis(out.values, -1, 0), uo)


@pytest.mark.parametrize("kind", ["aligned", "scalar"])
def test_periodic_self_exchange_through_nccl(gpu_ctx, nccl_ctx, kind):
    """NCCL point-to-point on one GPU: a periodic axis 0 on a single rank with
    ghost planes (DeviceGrid force_ghosts) gets its wrap through the halo
    exchange -- ncclSend/ncclRecv to itself, both neighbours the same rank,
    every stage -- and must reproduce the in-kernel wrap bitwise."""
    n = (12, 16, 32)
    cs = [np.arange(m, dtype=float) * h for m, h in zip(n, (0.3, 0.2, 0.1))]
    from paper_2403_01004_b200 import mesh
    grid = mesh.build_grid(list(n), coords=cs)
    per = mesh.FaceBC("periodic")
    bc = mesh.BoundaryCondition(((per, per), (mesh.FaceBC("neumann"), mesh.FaceBC("neumann")), (per, per)))
    rng = np.random.default_rng(5)
    u = operators.Field(grid, rng.uniform(0.5, 2.0, size=n + (1,)))
    if kind == "aligned":
        b = rng.normal(size=n + (3,))
        b /= np.linalg.norm(b, axis=-1, keepdims=True)
        make = lambda: operators.DiffusionOperator.aligned(  # noqa: E731
            operators.AlignedConductionConfig(b_hat=b, bc=bc), u)
    else:
        make = lambda: operators.DiffusionOperator.scalar(  # noqa: E731
            operators.ScalarDiffusionConfig(nu=1.0, bc=bc), 1)
    dg = device.DeviceGrid(grid, bc, nccl_ctx, force_ghosts=True)
    assert dg.ghost_lo and dg.ghost_hi
    nccl_ctx._grids[(id(grid), id(bc))] = (grid, bc, dg)
    res = []
    for ctx in (gpu_ctx, nccl_ctx):
        op = make()
        dtE = op.device_op(grid, 1, ctx).dt_euler
        out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), u, 40 * dtE, ctx=ctx)
        res.append((dtE, [e.iters for e in rep.entries], out.values.copy()))
    assert res[0][0] == res[1][0]
    assert res[0][1] == res[1][1]
    assert np.array_equal(res[0][2], res[1][2])


@pytest.mark.parametrize("name", ["aligned", "scalar", "viscous"])
def test_pcg_split_reduction_bitwise_equals_single_rank(gpu_ctx, nccl_ctx, name):
    """The r-slab PCG reduction (per-plane sums -> ncclAllReduce of the
    per-plane vector -> k_pcg_fin's fixed-order sum over the global planes)
    is bitwise the single-rank reduction: same iteration counts, same field
    bits -- the GPU-count invariance of SURVEY.md §8e on the device."""
    if name == "aligned":
        w = configs.c4(n=(24, 40, 64))
        cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
        u = operators.Field(w.grid, w.fields["T"])
        make = lambda: operators.DiffusionOperator.aligned(cfg, u)  # noqa: E731
        nc = 1
    elif name == "scalar":
        w = configs.c1(n=(20, 16, 32))
        cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc)
        u = operators.Field(w.grid, w.fields["u"][..., None])
        make = lambda: operators.DiffusionOperator.scalar(cfg, 1)  # noqa: E731
        nc = 1
    else:
        w = configs.c2(n=(20, 16, 32))
        cfg = operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc, vector_metric=True)
        u = operators.Field(w.grid, w.fields["v"])
        make = lambda: operators.DiffusionOperator.scalar(cfg, 3)  # noqa: E731
        nc = 3
    res = []
    for ctx in (gpu_ctx, nccl_ctx):
        op = make()
        dtE = op.device_op(w.grid, nc, ctx).dt_euler
        out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("backward_euler", tol=1e-9), u, 500 * dtE, ctx=ctx)
        res.append(([e.iters for e in rep.entries], [e.relres for e in rep.entries], out.values.copy()))
    assert sum(res[0][0]) > 10
    assert res[0][0] == res[1][0]
    assert res[0][1] == res[1][1]
    assert np.array_equal(res[0][2], res[1][2])
