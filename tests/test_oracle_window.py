"""The window restriction used by the full-size GPU checks
(tests/test_gpu_fullsize.py) reproduces the full-domain oracle bit for bit on
every plane far enough from the window edges (CPU only)."""
import numpy as np

from helpers import oracle_aligned, oracle_geometry, soa, window_geometry
from oracle import operators as oops
from oracle import ptl as optl
from oracle import schemes as osch
from paper_2403_01004_b200 import configs


def test_window_apply_and_stages_match_full_domain():
    w = configs.c5(n=(24, 16, 32), host=True)
    full = oracle_aligned(w.grid, w.bc, w.fields["b"], w.fields["T"], rho=w.fields["rho"])
    u = soa(w.fields["T"][..., None])
    F = full.apply(u)
    s, dt = 3, 1e-7
    us = osch.sts_step(full.apply, u, F, dt, s, "rkl2", full.geom.pinned)
    geom = oracle_geometry(w.grid, w.bc)
    for a, b in [(0, 3), (10, 13), (21, 24)]:
        lo, hi = max(a - s - 1, 0), min(b + s + 1, 24)
        gw = window_geometry(geom, lo, hi)
        T = configs.temperature(w.grid, w.seed, i0=lo, n0=hi - lo)
        assert np.array_equal(T, w.fields["T"][lo:hi])
        bh = configs.dipole_bhat(w.grid, w.seed, i0=lo, n0=hi - lo)
        c = oops.aligned_coefficient(T, 1.0, None, 1e-10)
        op = optl.OracleOperator(gw, "aligned", 1, None, w.fields["rho"][lo:hi], False, soa(bh), c, 1.0)
        Fw = op.apply(T[None])
        assert np.array_equal(Fw[:, a - lo:b - lo], F[:, a:b])
        uw = osch.sts_step(op.apply, T[None], Fw, dt, s, "rkl2", op.geom.pinned)
        assert np.array_equal(uw[:, a - lo:b - lo], us[:, a:b])


def test_window_viscous_matches_full_domain():
    w = configs.c5(n=(12, 16, 32), host=True)
    geom = oracle_geometry(w.grid, w.bc)
    r3 = w.fields["rho"]
    full = optl.OracleOperator(geom, "scalar", 3, np.full(r3.shape, 1.0) * r3, r3, True)
    F = full.apply(soa(w.fields["v"]))
    for a, b in [(0, 3), (5, 8), (9, 12)]:
        lo, hi = max(a - 1, 0), min(b + 1, 12)
        gw = window_geometry(geom, lo, hi)
        rw = r3[lo:hi]
        op = optl.OracleOperator(gw, "scalar", 3, np.full(rw.shape, 1.0) * rw, rw, True)
        vw = soa(configs.harmonic_velocity(w.grid, w.seed, i0=lo, n0=hi - lo))
        assert np.array_equal(op.apply(vw)[:, a - lo:b - lo], F[:, a:b])
