"""The r-line preconditioner (PC2 substitute) on the CPU oracle: the Thomas
solve inverts the r-line block of A exactly, BE+PCG with it converges to the
dense solution and needs fewer iterations than point Jacobi on a radially
stretched Spitzer problem."""
import numpy as np

from helpers import oracle_aligned, soa
from oracle import operators as oops
from oracle import ptl as optl
from oracle import schemes as osch
from paper_2403_01004_b200 import configs


def _op(n=(16, 8, 16)):
    w = configs.c3(n=n)
    return w, oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"])


def test_line_solve_inverts_the_line_block():
    w, op = _op()
    _, dg = op.bound_and_diag()
    jl, ju = op.line_offdiag()
    dt = 50 * op.euler_dt()
    inv, cp = oops.line_factor(1.0, dg[0], jl, ju, dt)
    rng = np.random.default_rng(0)
    r = rng.normal(size=dg[0].shape)
    r[op.geom.pinned] = 0.0
    z = oops.line_solve(r, jl, inv, cp, dt)
    n0 = r.shape[0]
    m = 1.0 + dt * dg[0]
    Mz = m * z
    Mz[1:] += (dt * jl[1:]) * z[:-1]
    Mz[:-1] += (dt * ju[:-1]) * z[1:]
    assert np.max(np.abs(Mz - r)) <= 1e-12 * np.max(np.abs(r))
    assert np.all(z[op.geom.pinned] == 0.0)
    assert n0 == 16


def test_line_offdiag_is_the_operator_coupling():
    """-J_{i,i+1} from the Hessian rows equals -dF_i/dT_{i+1} probed on the operator."""
    w, op = _op((8, 6, 8))
    jl, ju = op.line_offdiag()
    i, j, k = 4, 3, 5
    e = np.zeros((1,) + op.geom.shape)
    e[0, i + 1, j, k] = 1.0
    assert np.isclose(-op.apply(e)[0, i, j, k], ju[i, j, k], rtol=1e-12, atol=0)
    e[:] = 0.0
    e[0, i - 1, j, k] = 1.0
    assert np.isclose(-op.apply(e)[0, i, j, k], jl[i, j, k], rtol=1e-12, atol=0)


def test_line_pcg_converges_with_fewer_iterations():
    w, op = _op((24, 8, 16))
    u = soa(w.fields["T"][..., None])
    dtE = op.euler_dt()
    out = {}
    for pc in ("jacobi", "line-r"):
        uo, rep = optl.cycle_operator(op, optl.OracleScheme("backward_euler", tol=1e-10, preconditioner=pc),
                                      u, 1e3 * dtE, use_ptl=False, dt_euler=dtE)
        out[pc] = (uo, rep[0].iters)
    a, b = out["jacobi"][0], out["line-r"][0]
    assert np.linalg.norm(a - b) <= 1e-8 * np.linalg.norm(a)
    assert out["line-r"][1] < out["jacobi"][1]
