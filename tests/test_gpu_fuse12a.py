"""The fused stage-1+2 launch of the aligned TMA march (EpiStageA12: u1 = u0 +
mt1 y0 formed in the input slot as each plane lands, F(u1) and u2 in the same
pass, u1 written only when stage 3 follows) against the two-launch path
(PC_NO_FUSE12A: k_stage1 + k_aligned_tma<EpiStage>) and the oracle: identical
bits, stage counts and blow-up stages.  The grids take the TMA march
(n2 % 32 == 0) with partial theta tiles and Dirichlet (pinned) r ends; the
densities cover no rho, a radial rho (one value per plane) and a 3-D rho."""
import numpy as np
import pytest

from helpers import oracle_aligned, soa
from oracle import ptl as optl
from oracle import schemes as osch
from paper_2403_01004_b200 import configs, errors, mesh, operators, ptl, schemes

pytestmark = pytest.mark.gpu


def _case(rho_kind, n=(20, 40, 64)):
    w = configs.c3(n=n)
    rho = None
    if rho_kind != "none":
        r = np.asarray(w.grid.coords[0])
        rho = np.broadcast_to(np.exp(-10.0 * (r - 1.0))[:, None, None], tuple(w.grid.shape)).copy()
        if rho_kind == "field":
            rho *= 1.0 + 0.1 * np.random.default_rng(5).random(rho.shape)
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc, rho=rho)
    op = operators.DiffusionOperator.aligned(cfg, operators.Field(w.grid, w.fields["T"]))
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"], rho=rho)
    return w, op, oop


def _both(monkeypatch, run):
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("PC_NO_FUSE12A", env)
        else:
            monkeypatch.delenv("PC_NO_FUSE12A", raising=False)
        outs.append(run())
    monkeypatch.delenv("PC_NO_FUSE12A", raising=False)
    return outs


@pytest.mark.parametrize("rho_kind", ["none", "radial", "field"])
def test_fused_cycle_bitwise_with_two_launch_path_and_oracle(gpu_ctx, monkeypatch, rho_kind):
    """PTL cycles and an unlimited cycle (s >= 3: u1 written for stage 3)."""
    w, op, oop = _case(rho_kind)
    dtE = op.device_op(w.grid, 1).dt_euler
    assert dtE == oop.euler_dt()
    T = w.fields["T"]
    for use_ptl, ratio in ((True, 1e4), (False, 60.0)):
        def run():
            o, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), mesh.Field(w.grid, T), ratio * dtE,
                                        ptl.PtlConfig(enabled=use_ptl))
            return o.values.copy(), [(e.iters, e.dt) for e in rep.entries]
        a, b = _both(monkeypatch, run)
        assert a[1] == b[1]
        assert np.array_equal(a[0], b[0])
        assert a[0].tobytes() == b[0].tobytes()  # signed zeros too
        uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(T[..., None]), ratio * dtE,
                                       dt_euler=dtE, use_ptl=use_ptl)
        assert [it for it, _ in a[1]] == [r.iters for r in repo]
        assert [dt for _, dt in a[1]] == [r.dt for r in repo]
        assert np.array_equal(a[0][..., 0], uo[0])
        if not use_ptl:
            assert a[1][0][0] >= 3  # the u1-writing variant ran


def test_fused_step_rkl2_rkg2_s2_to_s5(gpu_ctx, monkeypatch):
    """pc_step_sts (schemes.step_*) with s = 2..5: both paths and the oracle bit for bit."""
    w, op, oop = _case("radial", n=(18, 24, 32))
    dtE = oop.euler_dt()
    T = w.fields["T"]
    for kind, step in (("rkl2", schemes.step_rkl2), ("rkg2", schemes.step_rkg2)):
        for r in (1.0, 3.0, 12.0):
            dt = r * dtE
            a, b = _both(monkeypatch, lambda: step(op, mesh.Field(w.grid, T), dt, dtE).values.copy())
            assert a.tobytes() == b.tobytes(), (kind, r)
            s = (osch.rkl2_iteration_count if kind == "rkl2" else osch.rkg2_iteration_count)(dt, dtE)
            u0 = soa(T[..., None])
            uo = osch.sts_step(oop.apply, u0, oop.apply(u0), dt, s, kind, oop.geom.pinned)
            assert np.array_equal(a[..., 0], uo[0]), (kind, r, s)


@pytest.mark.parametrize("r", [1.0, 2.0])
def test_fused_blowup_names_stage_one(gpu_ctx, monkeypatch, r):
    """A non-finite u1 (formed in shared memory, stored only when s >= 3)
    reports stage 1 on both paths, as the oracle does.  r = 1: s = 2; r = 2: s = 3."""
    w, op, oop = _case("none", n=(14, 20, 32))
    dtE = oop.euler_dt()
    T = w.fields["T"].copy()
    T[7, 9, 16] = 1.7e308  # F overflows at the neighbours; u1 = u0 + mt1 y0 is non-finite
    u0 = soa(T[..., None])
    with np.errstate(all="ignore"), pytest.raises(osch.BlowUpError) as eo:
        osch.sts_step(oop.apply, u0, oop.apply(u0), r * dtE, osch.rkl2_iteration_count(r * dtE, dtE), "rkl2",
                      oop.geom.pinned)
    assert eo.value.stage == 1

    def run():
        with pytest.raises(errors.BlowUpError) as ei:
            schemes.step_rkl2(op, mesh.Field(w.grid, T), r * dtE, dtE)
        return ei.value.stage
    assert _both(monkeypatch, run) == [1, 1]


def test_fused_launch_counted(gpu_ctx, monkeypatch):
    """The fused launch is what runs (its own hot-loop kind), and the two-launch path when it is switched off."""
    from paper_2403_01004_b200 import device
    w, op, oop = _case("none", n=(18, 24, 32))
    dtE = oop.euler_dt()
    ctx = device.default_context()
    counts = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("PC_NO_FUSE12A", env)
        ctx.enable_timing(True)
        ctx.reset_stats()
        schemes.step_rkl2(op, mesh.Field(w.grid, w.fields["T"]), 12.0 * dtE, dtE)
        k = ctx.stats_by_kind()
        ctx.enable_timing(False)
        counts.append((k["sts_af12"]["launches"] + k["sts_af12w"]["launches"], k["sts_aligned"]["launches"]))
    monkeypatch.delenv("PC_NO_FUSE12A", raising=False)
    s = osch.rkl2_iteration_count(12.0 * dtE, dtE)
    assert counts == [(1, s - 2), (0, s - 1)]
