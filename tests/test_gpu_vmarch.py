"""The vector march (k_vec_march, csrc/vmarch.cuh) -- y0 = F(u0) + argmax and
the fused stages 1 + 2 of the 3-component spherical viscosity operator --
against k_scalar_march (PC_NO_VMARCH=1) and the oracle: identical bits, stage
counts and PTL reports.  PC_VMARCH_STRICT=1 makes a vector launch that would
silently fall back to k_scalar_march an error, so the default leg provably
ran the new kernel.  Grids cover: several r-chunks with a partial last one
(PC_SMARCH_R), theta extents that are not a multiple of the 8-row tile, one
and several 32-column phi tiles (the periodic seam strips), Dirichlet r-ends,
and the four D modes (constant nu, nu field, nu rho with a 3-D rho, nu rho with
a radial rho read once per plane)."""
import numpy as np
import pytest

from helpers import oracle_scalar, soa
from oracle import ptl as optl
from oracle import schemes as osch
from paper_2403_01004_b200 import configs, mesh, operators, ptl, schemes

pytestmark = pytest.mark.gpu


def _op(w, kind):
    v = w.fields["v"]
    shape = tuple(w.grid.shape)
    if kind == "const":
        return (operators.DiffusionOperator.scalar(
                    operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc, vector_metric=True), 3),
                oracle_scalar(w.grid, w.bc, ncomp=3, vector_metric=True), v)
    if kind == "nu_field":
        nu = np.random.default_rng(7).uniform(0.5, 2.0, shape)
        return (operators.DiffusionOperator.scalar(
                    operators.ScalarDiffusionConfig(nu=nu, bc=w.bc, vector_metric=True), 3),
                oracle_scalar(w.grid, w.bc, nu=nu, ncomp=3, vector_metric=True), v)
    r = np.asarray(w.grid.coords[0])
    rho = np.broadcast_to(np.exp(-10.0 * (r - 1.0))[:, None, None], shape).copy()
    if kind != "rho_radial":  # (radial: C5's density, read per plane -- DM 3)
        rho *= 1.0 + 0.1 * np.random.default_rng(5).random(shape)
    return (operators.DiffusionOperator.scalar(
                operators.ScalarDiffusionConfig(nu=1.0, rho=rho, bc=w.bc, vector_metric=True), 3),
            oracle_scalar(w.grid, w.bc, rho=rho, ncomp=3, vector_metric=True), v)


def _run(monkeypatch, op, w, u, T, use_ptl, vm):
    if vm:
        monkeypatch.delenv("PC_NO_VMARCH", raising=False)
        monkeypatch.setenv("PC_VMARCH_STRICT", "1")
    else:
        monkeypatch.setenv("PC_NO_VMARCH", "1")
    o, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), mesh.Field(w.grid, u), T,
                                ptl.PtlConfig(enabled=use_ptl))
    monkeypatch.delenv("PC_VMARCH_STRICT", raising=False)
    monkeypatch.delenv("PC_NO_VMARCH", raising=False)
    return o.values.copy(), [(e.iters, e.dt, e.limited) for e in rep.entries]


CASES = [((20, 24, 32), "const", None), ((21, 20, 64), "rho", "8"), ((37, 12, 96), "nu_field", "8"),
         ((18, 16, 32), "rho", "4"), ((27, 20, 64), "rho_radial", "8")]


@pytest.mark.parametrize("n,kind,R", CASES)
def test_vmarch_cycle_bitwise_with_scalar_march_and_oracle(gpu_ctx, monkeypatch, n, kind, R):
    """PTL cycles (s = 2: F+argmax + the fused stage 1+2 launch) and an
    unlimited cycle (s >= 3: u1 written) on the host-driven loop."""
    monkeypatch.setenv("PC_NO_PERSIST", "1")
    if R:
        monkeypatch.setenv("PC_SMARCH_R", R)
    w = configs.c2(n=n)
    op, oop, u = _op(w, kind)
    dtE = op.device_op(w.grid, 3).dt_euler
    assert dtE == oop.euler_dt()
    for use_ptl in (True, False):
        a = _run(monkeypatch, op, w, u, 300 * dtE, use_ptl, True)
        b = _run(monkeypatch, op, w, u, 300 * dtE, use_ptl, False)
        assert a[1] == b[1]
        assert np.array_equal(a[0], b[0])
        uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(u), 300 * dtE, dt_euler=dtE,
                                       use_ptl=use_ptl)
        assert [it for it, _, _ in a[1]] == [r.iters for r in repo]
        assert np.array_equal(np.moveaxis(a[0], -1, 0), uo)
        if not use_ptl:
            assert a[1][0][0] >= 3


def test_vmarch_argmax_ties_and_index(gpu_ctx, monkeypatch):
    """A field whose |F| maximum is reached at many nodes (a mirrored impulse
    pattern): the argmax reported to PTL is the lowest AoS index, as the
    oracle's np.argmax -- the cycle reports agree bit for bit."""
    monkeypatch.setenv("PC_NO_PERSIST", "1")
    w = configs.c2(n=(16, 16, 64))
    op, oop, _ = _op(w, "const")
    u = np.zeros(tuple(w.grid.shape) + (3,))
    u[8, 5, 3, 1] = 1.0
    u[8, 5, 35, 1] = 1.0   # the same |F| pattern one phi tile over
    u[8, 10, 3, 1] = 1.0   # mirrored theta row: equal |F| only if the metric is symmetric
    dtE = oop.euler_dt()
    a = _run(monkeypatch, op, w, u, 50 * dtE, True, True)
    b = _run(monkeypatch, op, w, u, 50 * dtE, True, False)
    assert a[1] == b[1] and np.array_equal(a[0], b[0])
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(u), 50 * dtE, dt_euler=dtE, use_ptl=True)
    assert [it for it, _, _ in a[1]] == [r.iters for r in repo]
    assert np.array_equal(np.moveaxis(a[0], -1, 0), uo)


def test_vmarch_radial_rho_equals_field_path(gpu_ctx, monkeypatch):
    """A radial density read once per plane (DM 3) gives the bits of the
    staged-rho path (PC_NO_RADIAL_RHO=1 at freeze) and the oracle."""
    monkeypatch.setenv("PC_NO_PERSIST", "1")
    monkeypatch.setenv("PC_SMARCH_R", "8")
    w = configs.c2(n=(27, 20, 64))
    outs = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("PC_NO_RADIAL_RHO", env)
        else:
            monkeypatch.delenv("PC_NO_RADIAL_RHO", raising=False)
        op, oop, u = _op(w, "rho_radial")  # (the detection runs when the operator freezes)
        dtE = op.device_op(w.grid, 3).dt_euler
        outs.append(_run(monkeypatch, op, w, u, 300 * dtE, True, True))
    monkeypatch.delenv("PC_NO_RADIAL_RHO", raising=False)
    assert outs[0][1] == outs[1][1] and np.array_equal(outs[0][0], outs[1][0])
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("rkl2"), soa(u), 300 * dtE, dt_euler=dtE, use_ptl=True)
    assert [it for it, _, _ in outs[0][1]] == [r.iters for r in repo]
    assert np.array_equal(np.moveaxis(outs[0][0], -1, 0), uo)


@pytest.mark.parametrize("kind", ["const", "rho", "rho_radial"])
def test_vmarch_fused_step_sts(gpu_ctx, monkeypatch, kind):
    """schemes.step_rkl2 / step_rkg2 (s = 2..5, fused stage 1+2 on the new
    kernel) equal the oracle bit for bit."""
    monkeypatch.setenv("PC_VMARCH_STRICT", "1")
    w = configs.c2(n=(14, 20, 64))
    op, oop, v = _op(w, kind)
    dtE = oop.euler_dt()
    for name, step in (("rkl2", schemes.step_rkl2), ("rkg2", schemes.step_rkg2)):
        for r in (1.0, 3.0, 12.0):
            dt = r * dtE
            out = step(op, mesh.Field(w.grid, v), dt, dtE)
            s = (osch.rkl2_iteration_count if name == "rkl2" else osch.rkg2_iteration_count)(dt, dtE)
            u0 = soa(v)
            uo = osch.sts_step(oop.apply, u0, oop.apply(u0), dt, s, name, oop.geom.pinned)
            assert np.array_equal(np.moveaxis(out.values, -1, 0), uo), (name, r, s)
