"""analysis on the production GPU path: amplification
factors measured from one device step of each scheme agree with the closed
forms (two evaluations agree; BE to the PCG tolerance), the
fitted convergence orders, the fine-Euler reference."""
import math

import numpy as np
import pytest

from paper_2403_01004_b200 import analysis, cli, mesh, operators

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,r,tol", [("rkl2", 500, 1e-11), ("rkg2", 500, 1e-11), ("euler", 0.9, 1e-12),
                                        ("be", 500, 1e-10), ("rkg2", 20, 1e-12)])
def test_amplification_two_ways(gpu_ctx, kind, r, tol):
    theta, run = analysis.amplification_run(kind, r)
    closed = analysis.amplification(kind, r, theta)
    assert np.max(np.abs(run - closed)) <= tol
    assert len(theta) == 512 and theta[-1] == math.pi


@pytest.mark.parametrize("kind,order", [("be", 1.0), ("rkg2", 2.0), ("rkl2", 2.0), ("euler", 1.0)])
def test_convergence_orders(gpu_ctx, kind, order):
    slope, dts, errs = analysis.convergence_study(kind)
    assert abs(slope - order) <= 0.1, (slope, errs)


def test_convergence_cli(gpu_ctx, capsys):
    assert cli.main(["convergence", "--scheme", "be", "--problem", "sine"]) == 0
    out = capsys.readouterr().out
    assert "be: fitted order" in out and abs(float(out.split()[-1]) - 1.0) < 0.1


def test_fine_euler_reference(gpu_ctx):
    """F = 0 -> identity; a single Fourier mode decays as the analytic e^{-lam t} to 1e-6 at n_sub = 1e4."""
    g, op = analysis._periodic_problem(16)
    n = 32
    u0 = np.sin(math.pi * 2 * np.arange(n) / 16)
    lam = 4.0 * math.sin(math.pi * 2 / 16 / 2) ** 2
    T = 0.5
    out = analysis.oracle_fine_euler(op, mesh.Field(g, u0[:, None]), T, 10000)
    assert np.max(np.abs(out.values[:, 0] - math.exp(-lam * T) * u0)) <= 1e-6
    bc = mesh.BoundaryCondition.periodic(1)
    zero = operators.DiffusionOperator.scalar(operators.ScalarDiffusionConfig(nu=0.0, bc=bc), 1)
    f = mesh.Field(g, u0[:, None])
    with pytest.raises(ValueError):
        analysis.oracle_fine_euler(op, f, 2.0, 2)  # substep 1.0 above the explicit limit 0.5
    assert np.array_equal(analysis.oracle_fine_euler(zero, f, T, 7).values, f.values)
