"""C1 (48x48x96 spherical scalar diffusion) parity: GPU path vs CPU oracle.

Contract (BASELINE.json north star): identical PTL cycle counts, stage / PCG
iteration counts, and final fields within relative L2 1e-10.  The RKL2 path
is elementwise, so it is checked BIT-FOR-BIT (cycle dts and the field).
"""
import numpy as np
import pytest

from helpers import oracle_scalar, soa
from oracle import ptl as optl
from paper_2403_01004_b200 import configs, operators, ptl, schemes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    return configs.c1()


def _op(w):
    return operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=1.0, bc=w.bc))


def test_c1_euler_dt_bitwise(gpu_ctx, c1):
    dtE = _op(c1).device_op(c1.grid, 1).dt_euler
    assert dtE == oracle_scalar(c1.grid, c1.bc).euler_dt()


def test_c1_apply_bitwise(gpu_ctx, c1):
    u = c1.fields["u"]
    F = operators.apply_scalar_diffusion(operators.Field(c1.grid, u), operators.ScalarDiffusionConfig(1.0, bc=c1.bc))
    Fo = oracle_scalar(c1.grid, c1.bc).apply(soa(u[..., None]))
    assert np.array_equal(F.values[..., 0], Fo[0])


@pytest.mark.parametrize("kind", ["rkl2", "rkg2"])
def test_c1_sts_ptl_parity(gpu_ctx, c1, kind):
    op = _op(c1)
    u = operators.Field(c1.grid, c1.fields["u"])
    dtE = op.device_op(c1.grid, 1).dt_euler
    out, rep = ptl.cycle_operator(op, schemes.SchemeConfig(kind), u, 500 * dtE, ptl.PtlConfig())
    oop = oracle_scalar(c1.grid, c1.bc)
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme(kind), soa(c1.fields["u"][..., None]), 500 * dtE, dt_euler=dtE)
    assert rep.n_cycles == len(repo)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    assert [e.dt for e in rep.entries] == [r.dt for r in repo]
    assert np.array_equal(out.values[..., 0], uo[0])


def test_c1_be_pcg_ptl_parity(gpu_ctx, c1):
    op = _op(c1)
    u = operators.Field(c1.grid, c1.fields["u"])
    dtE = op.device_op(c1.grid, 1).dt_euler
    sc = schemes.SchemeConfig("backward_euler", tol=1e-10)
    out, rep = ptl.cycle_operator(op, sc, u, 500 * dtE, ptl.PtlConfig())
    oop = oracle_scalar(c1.grid, c1.bc)
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("backward_euler", tol=1e-10),
                                   soa(c1.fields["u"][..., None]), 500 * dtE, dt_euler=dtE)
    assert rep.n_cycles == len(repo)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    a, b = out.values[..., 0], uo[0]
    assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-10
