"""cli run: config validation on CPU (an invalid config
exits 2 with a line-anchored message, before any device work)."""
import os

import pytest

from paper_2403_01004_b200 import cli

GOOD = """[grid]
metric = cartesian
sizes = 11
extents = 0, 1
bc = dirichlet:0

[operator.d]
kind = scalar
field = u

[initial]
u = step

[run]
outer_dt = 0.01
"""


def _run(tmp_path, text, capsys):
    p = tmp_path / "x.cfg"
    p.write_text(text)
    rc = cli.main(["run", str(p)])
    return rc, capsys.readouterr().err


@pytest.mark.parametrize("edit,line,msg", [
    (("[run]", "[runn]"), 14, "unknown section"),
    (("kind = scalar", "kind = scalar\ncolour = red"), 9, "unknown key"),
    (("sizes = 11", "sizes = eleven"), 3, "bad value"),
    (("kind = scalar", "kind = nonlinear"), 8, "unknown operator kind"),
    (("u = step", "u = random"), 12, "seed is mandatory"),
    (("bc = dirichlet:0", "bc = robin"), 5, "bad value"),
    (("outer_dt = 0.01", "outer_dt = 0.01\ndt_over_dt_euler = 5"), 14, "exactly one"),
])
def test_invalid_config_is_line_anchored(tmp_path, capsys, edit, line, msg):
    rc, err = _run(tmp_path, GOOD.replace(*edit), capsys)
    assert rc == 2
    assert f"x.cfg:{line}:" in err and msg in err, err


def test_usage_error(capsys):
    assert cli.main(["frobnicate"]) == 2
    assert "usage" in capsys.readouterr().err
    assert cli.main(["run"]) == 2


def test_shipped_examples_parse():
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples")
    for f in sorted(os.listdir(root)):
        c = cli._Cfg(os.path.join(root, f))
        grid, bc = cli.build_grid(c)
        assert grid.npoints > 0


def test_analysis_usage_errors(capsys, tmp_path):
    assert cli.main(["ampfactor", "--schemes", "", "--r", "500", "--out", str(tmp_path / "a.csv")]) == 2
    assert cli.main(["speedup", "--rmin", "10", "--rmax", "1", "--out", str(tmp_path / "s.csv")]) == 2
    assert cli.main(["convergence", "--scheme", "rkg2", "--problem", "square"]) == 2
    assert "usage error" in capsys.readouterr().err
