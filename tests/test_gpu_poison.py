"""Substitutes for compute-sanitizer (closed on this GPU pool, see
profiles/r02_sanitizer_closed.txt): every kernel family of
scripts/sanitize_cases.py -- TMA march, cp.async march, 7-point march,
persistent loop, PCG (Jacobi, r-line), the split overlap schedule -- runs

* with PC_POISON=1: every workspace buffer is handed out filled with NaN
  bytes, so a read of memory the kernels did not write first shows up as a
  NaN / parity failure (the initcheck substitute);
* three times in one process: every run must stay bitwise on the oracle (a
  shared-memory or mbarrier race shows up as run-to-run differences)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("poison", [True, False], ids=["poison", "plain"])
def test_kernel_families_poisoned_and_repeated(poison):
    env = dict(os.environ)
    if poison:
        env["PC_POISON"] = "1"
    cases = ["tma", "cpasync", "smarch", "persist", "pcg", "split"] * (1 if poison else 3)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py")] + cases,
                       capture_output=True, text=True, env=env, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "all cases ok" in r.stdout


def test_smarch_tma_staging_opt_in():
    """The opt-in TMA staging of the 7-point march (PC_SMARCH_TMA=1) is
    bitwise the cp.async staging and the oracle (smarch and persist cases)."""
    env = dict(os.environ, PC_SMARCH_TMA="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py"), "smarch", "pcg"],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
