"""The fused stage-1+2 launch of the 7-point march (SEpiStage12: u1 = u0 +
mt1 y0 formed in shared memory, F(u1) and u2 in the same pass, u1 written only
when stage 3 follows) against the two-launch path (PC_NO_FUSE12) and the
oracle: identical bits, stage counts and blow-up stages.  PC_NO_PERSIST keeps
the small test grids on the host-driven cycle loop (sts_stages), the path the
C2-size grids take."""
import numpy as np
import pytest

from helpers import oracle_scalar, soa
from oracle import ptl as optl
from oracle import schemes as osch
from paper_2403_01004_b200 import configs, errors, mesh, operators, ptl, schemes

pytestmark = pytest.mark.gpu


def _ops(w, kind):
    """(device operator, oracle operator, state array, ncomp) of a test case."""
    if kind == "scalar":
        u = w.fields["u"][..., None]
        return (operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc), 1),
                oracle_scalar(w.grid, w.bc), u, 1)
    if kind == "scalar_D":
        rng = np.random.default_rng(11)
        nu = rng.uniform(0.5, 2.0, tuple(w.grid.shape))
        u = w.fields["u"][..., None]
        return (operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=nu, bc=w.bc), 1),
                oracle_scalar(w.grid, w.bc, nu=nu), u, 1)
    v = w.fields["v"]
    if kind == "vector":
        return (operators.DiffusionOperator.scalar(
                    operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc, vector_metric=True), 3),
                oracle_scalar(w.grid, w.bc, ncomp=3, vector_metric=True), v, 3)
    r = np.asarray(w.grid.coords[0])
    rho = np.broadcast_to(np.exp(-10.0 * (r - 1.0))[:, None, None], tuple(w.grid.shape)).copy()
    rho *= 1.0 + 0.1 * np.random.default_rng(5).random(rho.shape)  # a true 3-D density
    return (operators.DiffusionOperator.scalar(
                operators.ScalarDiffusionConfig(nu=1.0, rho=rho, bc=w.bc, vector_metric=True), 3),
            oracle_scalar(w.grid, w.bc, rho=rho, ncomp=3, vector_metric=True), v, 3)


def _case(kind):
    if kind in ("scalar", "scalar_D"):
        return configs.c1(n=(20, 24, 48))
    return configs.c2(n=(20, 24, 48))


@pytest.mark.parametrize("kind", ["scalar", "scalar_D", "vector", "vector_rho"])
def test_fused_cycle_bitwise_with_two_launch_path_and_oracle(gpu_ctx, monkeypatch, kind):
    """PTL cycles (mostly s = 2: no u1 write) and an unlimited cycle
    (s >= 3: u1 written for stage 3) through both paths and the oracle."""
    monkeypatch.setenv("PC_NO_PERSIST", "1")
    w = _case(kind)
    op, oop, u, nc = _ops(w, kind)
    dtE = op.device_op(w.grid, nc).dt_euler
    assert dtE == oop.euler_dt()
    for use_ptl in (True, False):
        outs = []
        for env in (None, "1"):
            if env:
                monkeypatch.setenv("PC_NO_FUSE12", env)
            else:
                monkeypatch.delenv("PC_NO_FUSE12", raising=False)
            o, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), mesh.Field(w.grid, u), 400 * dtE,
                                        ptl.PtlConfig(enabled=use_ptl))
            outs.append((o.values.copy(), [(e.iters, e.dt) for e in rep.entries]))
        monkeypatch.delenv("PC_NO_FUSE12", raising=False)
        assert outs[0][1] == outs[1][1]
        assert np.array_equal(outs[0][0], outs[1][0])
        uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(u), 400 * dtE, dt_euler=dtE,
                                       use_ptl=use_ptl)
        assert [it for it, _ in outs[0][1]] == [r.iters for r in repo]
        assert np.array_equal(np.moveaxis(outs[0][0], -1, 0), uo)
        if not use_ptl:
            assert outs[0][1][0][0] >= 3  # the u1-writing variant ran


def test_fused_step_rkg2_and_rkl2(gpu_ctx):
    """pc_step_sts (schemes.step_*) with s = 2..5 on the fused path equals the oracle bit for bit."""
    w = configs.c2(n=(16, 20, 40))
    op, oop, v, nc = _ops(w, "vector")
    dtE = oop.euler_dt()
    for kind, step in (("rkl2", schemes.step_rkl2), ("rkg2", schemes.step_rkg2)):
        for r in (1.0, 3.0, 12.0):
            dt = r * dtE
            out = step(op, mesh.Field(w.grid, v), dt, dtE)
            s = (osch.rkl2_iteration_count if kind == "rkl2" else osch.rkg2_iteration_count)(dt, dtE)
            u0 = soa(v)
            uo = osch.sts_step(oop.apply, u0, oop.apply(u0), dt, s, kind, oop.geom.pinned)
            assert np.array_equal(np.moveaxis(out.values, -1, 0), uo), (kind, r, s)


@pytest.mark.parametrize("r", [1.0, 2.0])
def test_fused_blowup_names_stage_one(gpu_ctx, monkeypatch, r):
    """A non-finite u1 (formed in shared memory, never stored when s = 2)
    still reports stage 1 -- the oracle's stage and the separate k_stage1
    launch's.  r = 1: s = 2 (no u1 write); r = 2: s = 3."""
    w = configs.c1(n=(12, 12, 24))
    op, oop, u, _ = _ops(w, "scalar")
    dtE = oop.euler_dt()
    u = u.copy()
    u[6, 6, 12, 0] = 1.7e308  # F overflows; u1 = u0 + mt1 y0 is non-finite
    u0 = soa(u)
    with np.errstate(all="ignore"), pytest.raises(osch.BlowUpError) as eo:
        osch.sts_step(oop.apply, u0, oop.apply(u0), r * dtE, osch.rkl2_iteration_count(r * dtE, dtE), "rkl2",
                      oop.geom.pinned)
    assert eo.value.stage == 1
    stages = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("PC_NO_FUSE12", env)
        with pytest.raises(errors.BlowUpError) as ei:
            schemes.step_rkl2(op, mesh.Field(w.grid, u), r * dtE, dtE)
        stages.append(ei.value.stage)
    assert stages == [1, 1]


@pytest.mark.parametrize("kind", ["scalar", "scalar_D", "vector", "vector_rho"])
def test_persistent_cycle_bitwise_with_fused_host_loop(gpu_ctx, monkeypatch, kind):
    """The persistent small-grid cycle kernel (separate stage-1 pass) and the
    host-driven loop with the fused stage-1+2 march (PC_NO_PERSIST): the same
    bits and reports as each other and as the oracle, with PTL (s = 2) and
    without (s >= 3)."""
    w = _case(kind)
    op, oop, u, nc = _ops(w, kind)
    dtE = op.device_op(w.grid, nc).dt_euler
    for use_ptl in (True, False):
        outs = []
        for env in (None, "1"):
            if env:
                monkeypatch.setenv("PC_NO_PERSIST", env)
            else:
                monkeypatch.delenv("PC_NO_PERSIST", raising=False)
            o, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), mesh.Field(w.grid, u), 300 * dtE,
                                        ptl.PtlConfig(enabled=use_ptl))
            outs.append((o.values.copy(), [(e.iters, e.dt, e.limited) for e in rep.entries]))
        assert outs[0][1] == outs[1][1]
        assert np.array_equal(outs[0][0], outs[1][0])
        uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(u), 300 * dtE, dt_euler=dtE,
                                       use_ptl=use_ptl)
        assert [it for it, _, _ in outs[0][1]] == [r.iters for r in repo]
        assert np.array_equal(np.moveaxis(outs[0][0], -1, 0), uo)
