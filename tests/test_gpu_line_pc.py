"""The r-line preconditioner (PC2 substitute) on the GPU against the oracle:
identical PTL cycles and PCG iteration counts, fields within 1e-10 relative L2
(dot products are reduced in a different order than numpy's), and far fewer
iterations than point Jacobi on the radially stretched Spitzer problem."""
import numpy as np
import pytest

from helpers import oracle_aligned, soa
from oracle import ptl as optl
from paper_2403_01004_b200 import configs, operators, ptl, schemes

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [(24, 40, 64), (20, 24, 48)], ids=["tma", "cpasync"])
def test_line_pcg_parity(gpu_ctx, n):
    w = configs.c3(n=n)
    cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
    T = operators.Field(w.grid, w.fields["T"])
    op = operators.DiffusionOperator.aligned(cfg, T)
    dtE = op.device_op(w.grid, 1).dt_euler
    oop = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])
    res = {}
    for pc in ("line-r", "jacobi"):
        out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("backward_euler", tol=1e-9, preconditioner=pc), T,
                                      1e4 * dtE)
        res[pc] = (out, rep)
    out, rep = res["line-r"]
    uo, repo = optl.cycle_operator(oop, optl.OracleScheme("backward_euler", tol=1e-9, preconditioner="line-r"),
                                   soa(w.fields["T"][..., None]), 1e4 * dtE, dt_euler=dtE)
    assert [e.iters for e in rep.entries] == [r.iters for r in repo]
    a, b = out.values[..., 0], uo[0]
    assert np.linalg.norm(a - b) <= 1e-10 * np.linalg.norm(b)
    assert rep.total_iters * 3 < res["jacobi"][1].total_iters
