"""cli run end to end on the GPU (SPEC.md:492-500 examples): zero operators
leave the state unchanged, two runs write byte-identical CSVs, the shipped
step-data PTL experiment reports >= 1 cycle per outer step with sum dt ==
outer_dt."""
import csv
import filecmp
import os
import shutil

import pytest

from paper_2403_01004_b200 import cli, mesh

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_zero_operators_is_identity(gpu_ctx, tmp_path, monkeypatch):
    monkeypatch.chdir(tmp_path)
    (tmp_path / "z.cfg").write_text("[grid]\nsizes = 9, 7\nextents = 0, 1; 0, 2\nbc = neumann\n"
                                    "[initial]\nu = sinusoid\nu.k = 3, 1\n[run]\nout_prefix = z\n")
    assert cli.main(["run", "z.cfg"]) == 0
    c = cli._Cfg("z.cfg")
    grid, _ = cli.build_grid(c)
    init = cli.initial_state(c, grid, {"u": 1})["u"]
    mesh.write_field_csv(init, "ref.csv")
    assert filecmp.cmp("z_u.csv", "ref.csv", shallow=False)


@pytest.mark.parametrize("cfg", ["step_ptl.cfg", "c1_spherical.cfg"])
def test_runs_are_byte_identical_and_reports_sum(gpu_ctx, tmp_path, monkeypatch, cfg):
    monkeypatch.chdir(tmp_path)
    shutil.copy(os.path.join(ROOT, "examples", cfg), cfg)
    outs = []
    for rnd in range(2):
        assert cli.main(["run", cfg]) == 0
        d = tmp_path / f"r{rnd}"
        d.mkdir()
        for f in os.listdir(tmp_path):
            if f.endswith(".csv"):
                shutil.move(str(tmp_path / f), str(d / f))
        outs.append(d)
    names = sorted(os.listdir(outs[0]))
    assert names and names == sorted(os.listdir(outs[1]))
    for n in names:
        assert filecmp.cmp(outs[0] / n, outs[1] / n, shallow=False), n
    rep = [n for n in names if n.endswith("report.csv")][0]
    rows = list(csv.DictReader(open(outs[0] / rep)))
    steps = sorted({int(r["outer_step"]) for r in rows})
    assert steps == list(range(len(steps))) and len(steps) >= 1
    sums = {s: sum(float(r["dt"]) for r in rows if int(r["outer_step"]) == s) for s in steps}
    counts = {s: sum(1 for r in rows if int(r["outer_step"]) == s) for s in steps}
    vals = list(sums.values())
    assert all(abs(v - vals[0]) <= 1e-12 * vals[0] for v in vals)  # every outer step covers outer_dt
    assert all(n >= 1 for n in counts.values())
    assert any(r["limited"] == "1" for r in rows)  # the PTL limited at least one cycle
