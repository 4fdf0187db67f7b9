"""analysis closed forms and the SPEC's Fig. 1 examples (CPU:
the coefficient tables come from the library's host entry points)."""
import math

import numpy as np

from paper_2403_01004_b200 import analysis, cli


def test_amplification_kats():
    assert math.isclose(analysis.amplification("be", 500, math.pi), 1.0 / 1001.0, rel_tol=1e-15)  # 9.990e-4
    assert math.isclose(analysis.exact_amplification(0.5, math.pi), math.exp(-1.0), rel_tol=1e-15)
    assert analysis.exact_amplification(500, math.pi) < 1e-300
    for k in ("be", "rkl2", "rkg2", "exact"):
        assert abs(analysis.amplification(k, 500, 1e-9) - 1.0) < 1e-9  # zero mode undamped


def test_speedup_kats():
    assert math.isclose(analysis.speedup_estimate("rkg2", 500), 500 / 55, rel_tol=1e-15)  # 9.09
    assert math.isclose(analysis.speedup_estimate("rkg2", 1), 1 / 3, rel_tol=1e-15)


def test_fig1_properties():
    th = math.pi * np.arange(1, 513) / 512
    be = analysis.amplification("be", 500, th)
    assert np.all(be > 0) and np.all(np.diff(be) < 0)  # BE positive, monotone decreasing
    hi = th >= math.pi / 2
    assert analysis.amplification("rkg2", 500, th)[hi].max() < analysis.amplification("rkl2", 500, th)[hi].max()
    for k in ("be", "rkl2", "rkg2"):  # unconditionally stable schemes over-estimate high-mode survival
        assert np.all(analysis.amplification(k, 500, th)[hi] >= analysis.exact_amplification(500, th)[hi])
        assert np.all(analysis.amplification(k, 500, th) <= 1.0 + 1e-12)


def test_ampfactor_csv(tmp_path):
    out = tmp_path / "amp.csv"
    assert cli.main(["ampfactor", "--schemes", "be,exact", "--r", "500", "--out", str(out)]) == 0
    rows = out.read_text().splitlines()
    assert rows[0] == "scheme,r,theta,amplification" and len(rows) == 1 + 2 * 512
    last_be = [r for r in rows if r.startswith("be,")][-1]
    assert math.isclose(float(last_be.split(",")[3]), 9.99000999000999e-4, rel_tol=1e-12)
