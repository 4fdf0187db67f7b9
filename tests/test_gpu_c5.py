"""C5 (coupled conduction + viscosity, rho = exp(-10 (r - 1))) at reduced size:
the device-generated inputs are bitwise the host recipes (configs.py), and one
split MAS step matches the oracle bit for bit (cycle and stage counts, both
fields)."""
import numpy as np
import pytest

from helpers import oracle_aligned, oracle_scalar, soa
from oracle import operators as oops
from oracle import ptl as optl
from paper_2403_01004_b200 import configs, device, operators, ptl, schemes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c5s():
    return configs.c5(n=(16, 20, 32), host=True)


def test_device_generation_bitwise(gpu_ctx, c5s):
    dg = device.device_grid(c5s.grid, c5s.bc, gpu_ctx)
    T = configs.gen_temperature(device.DeviceField(dg, 1), c5s.grid, c5s.seed)
    b = configs.gen_dipole(device.DeviceField(dg, 3), c5s.grid, c5s.seed)
    v = configs.gen_harmonic(device.DeviceField(dg, 3), c5s.grid, c5s.seed)
    rho = configs.gen_radial(device.DeviceField(dg, 1), c5s.meta["rho_r"])
    assert np.array_equal(T.download()[..., 0], c5s.fields["T"])
    assert np.array_equal(b.download(), c5s.fields["b"])
    assert np.array_equal(v.download(), c5s.fields["v"])
    assert np.array_equal(rho.download()[..., 0], c5s.fields["rho"])


def test_viscous_rho_field_apply_bitwise(gpu_ctx, c5s):
    rho = c5s.fields["rho"]
    cfg = operators.ScalarDiffusionConfig(nu=1.0, rho=rho, bc=c5s.bc, vector_metric=True)
    op = operators.DiffusionOperator.scalar(cfg, 3)
    v = operators.Field(c5s.grid, c5s.fields["v"])
    F = op.apply(v)
    oop = oracle_scalar(c5s.grid, c5s.bc, nu=1.0, rho=rho, ncomp=3, vector_metric=True)
    assert np.array_equal(np.moveaxis(F.values, -1, 0), oop.apply(soa(c5s.fields["v"])))
    assert op.device_op(c5s.grid, 3).dt_euler == oop.euler_dt()


def test_c5_split_step_parity(gpu_ctx, c5s):
    w = c5s
    dg = device.device_grid(w.grid, w.bc, gpu_ctx)
    rho_d = configs.gen_radial(device.DeviceField(dg, 1), w.meta["rho_r"])
    b_d = configs.gen_dipole(device.DeviceField(dg, 3), w.grid, w.seed)
    T_d = configs.gen_temperature(device.DeviceField(dg, 1), w.grid, w.seed)
    v_d = configs.gen_harmonic(device.DeviceField(dg, 3), w.grid, w.seed)
    cond = operators.DiffusionOperator.aligned(
        operators.AlignedConductionConfig(b_hat=b_d, rho=rho_d, m_p=3.0, k_B=1.0, bc=w.bc))
    visc = operators.DiffusionOperator.scalar(
        operators.ScalarDiffusionConfig(nu=1.0, rho=rho_d, bc=w.bc, vector_metric=True), 3)
    cond.freeze(T_d)
    dtE = min(cond.device_op(w.grid, 1).dt_euler, visc.device_op(w.grid, 3).dt_euler)
    outer = 200.0 * dtE
    sc = schemes.SchemeConfig("rkl2")
    state = ptl.split_advance([("T", cond), ("v", visc)], {"T": T_d, "v": v_d}, outer,
                                    [(sc, ptl.PtlConfig()), (sc, ptl.PtlConfig())])
    reps = state.reports
    # oracle
    oc = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"], rho=w.fields["rho"])
    ov = oracle_scalar(w.grid, w.bc, nu=1.0, rho=w.fields["rho"], ncomp=3, vector_metric=True)

    def refresh(op, st):
        op.c = oops.aligned_coefficient(st["T"][0])

    ost, oreps = optl.split_advance([("T", oc), ("v", ov)], {"T": soa(w.fields["T"][..., None]),
                                                             "v": soa(w.fields["v"])}, outer,
                                    [optl.OracleScheme("rkl2")] * 2, refresh=refresh)
    for rep, orep in zip(reps, oreps):
        assert [e.iters for e in rep.entries] == [r.iters for r in orep]
        assert [e.dt for e in rep.entries] == [r.dt for r in orep]
    assert np.array_equal(state["T"].download()[..., 0], ost["T"][0])
    assert np.array_equal(np.moveaxis(state["v"].download(), -1, 0), ost["v"])


def test_radial_rho_path_bitwise(gpu_ctx, c5s, monkeypatch):
    """A radial density is read per plane by the TMA march (no per-node rho
    stream); the field path (PC_NO_RADIAL_RHO) gives the same bits."""
    w = c5s
    T = operators.Field(w.grid, w.fields["T"])
    out = []
    for env in (None, "1"):
        if env:
            monkeypatch.setenv("PC_NO_RADIAL_RHO", env)
        cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], rho=w.fields["rho"], m_p=3.0, k_B=1.0, bc=w.bc)
        op = operators.DiffusionOperator.aligned(cfg, T)
        dtE = op.device_op(w.grid, 1).dt_euler
        o, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), T, 300 * dtE)
        out.append((o.values.copy(), [e.iters for e in rep.entries]))
    assert out[0][1] == out[1][1]
    assert np.array_equal(out[0][0], out[1][0])


def test_c5_split_step_host_fields_async_copies(gpu_ctx, c5s):
    """split_advance on HOST Fields (the e2e path): the second operator's state
    uploads on the copy stream while the first operator computes, and each
    state downloads as soon as its last operator is done.  Same bits and
    reports as the device-resident path and the oracle."""
    w = c5s
    T = operators.Field(w.grid, w.fields["T"])
    v = operators.Field(w.grid, w.fields["v"])
    pinned = [gpu_ctx.pin(a) for a in (w.fields["T"], w.fields["v"], w.fields["b"], w.fields["rho"])
              if a.flags.c_contiguous]  # page-locked: the copies really overlap
    try:
        _host_split_step(gpu_ctx, w, T, v)
    finally:
        for a in pinned:
            gpu_ctx.unpin(a)


def _host_split_step(gpu_ctx, w, T, v):
    cond = operators.DiffusionOperator.aligned(
        operators.AlignedConductionConfig(b_hat=w.fields["b"], rho=w.fields["rho"], m_p=3.0, k_B=1.0, bc=w.bc))
    visc = operators.DiffusionOperator.scalar(
        operators.ScalarDiffusionConfig(nu=1.0, rho=w.fields["rho"], bc=w.bc, vector_metric=True), 3)
    oc = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"], rho=w.fields["rho"])
    ov = oracle_scalar(w.grid, w.bc, nu=1.0, rho=w.fields["rho"], ncomp=3, vector_metric=True)
    dtE = min(oc.euler_dt(), ov.euler_dt())
    outer = 200.0 * dtE
    sc = schemes.SchemeConfig("rkl2")
    state = ptl.split_advance([("T", cond), ("v", visc)], {"T": T, "v": v}, outer,
                                    [(sc, ptl.PtlConfig()), (sc, ptl.PtlConfig())])
    reps = state.reports
    assert isinstance(state["T"], operators.Field) and isinstance(state["v"], operators.Field)

    def refresh(op, st):
        op.c = oops.aligned_coefficient(st["T"][0])

    ost, oreps = optl.split_advance([("T", oc), ("v", ov)], {"T": soa(w.fields["T"][..., None]),
                                                             "v": soa(w.fields["v"])}, outer,
                                    [optl.OracleScheme("rkl2")] * 2, refresh=refresh)
    for rep, orep in zip(reps, oreps):
        assert [e.iters for e in rep.entries] == [r.iters for r in orep]
    assert np.array_equal(state["T"].values[..., 0], ost["T"][0])
    assert np.array_equal(np.moveaxis(state["v"].values, -1, 0), ost["v"])


def test_async_upload_download_semantics(gpu_ctx, c5s):
    """upload_async: the next library call on the field waits for the copy on
    the device; download_async: valid after wait(); destroying a field with a
    copy in flight waits for it."""
    w = c5s
    dg = device.device_grid(w.grid, w.bc, gpu_ctx)
    v = device.pinned_empty(tuple(w.grid.shape) + (3,))
    v[...] = w.fields["v"]
    f = device.DeviceField(dg, 3).upload(v, async_=True)
    g = device.DeviceField(dg, 3).copy_from(f)  # waits for the upload on the device
    assert np.array_equal(g.download(), w.fields["v"])
    out = g.download_async()
    g.wait()
    assert np.array_equal(out, w.fields["v"])
    h = device.DeviceField(dg, 3).upload(v, async_=True)
    del h  # destroy with the copy possibly in flight
    cnt = f.count_failing(2)  # TEST_FINITE through a waited field
    assert cnt == 0
