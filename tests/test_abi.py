"""The C-ABI boundary without a GPU: the in-tree sm_100a library loads, exports
every entry point include/paracycle_b200.h declares (and the ctypes binding
binds exactly those), and its host-only functions -- the STS stage count and
coefficient tables, i.e. the integer decisions of schemes.step_rkl2 /
step_rkg2 -- agree bit for bit with the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import schemes as osch
from paper_2403_01004_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "paracycle_b200.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    build.build()  # no-op when up to date; nvcc cross-compiles without a GPU
    return _lib.lib()


def test_header_matches_binding():
    assert _declared() == sorted(_lib.EXPORTED)


def test_library_exports_every_declared_symbol(L):
    for name in _declared():
        assert hasattr(L, name), name
    assert L.pc_version() >= 1


def test_no_cuda_call_needed_for_host_entry_points(L):
    # error path: a bad argument is reported without touching the device
    assert L.pc_sts_table(_lib.RKL2, 1, 1.0, (ctypes.c_double * 5)()) == _lib.PC_E_INVALID
    assert "s >= 2" in _lib.last_error()
    assert L.pc_sts_table(_lib.RKG2, 4, 1.0, (ctypes.c_double * 20)()) == _lib.PC_E_INVALID


@pytest.mark.parametrize("ratio", [1e-9, 0.5, 1.0, 1.0000000001, 2.0, 7.3, 500.0, 2000.0, 1e4, 5e4, 123456.7])
def test_sts_counts_match_oracle(L, ratio):
    dtE = 3.7e-5
    dt = ratio * dtE
    assert L.pc_sts_count(_lib.RKL2, dt, dtE, 0) == osch.rkl2_iteration_count(dt, dtE)
    assert L.pc_sts_count(_lib.RKL2, dt, dtE, 1) == osch.rkl2_iteration_count(dt, dtE, True)
    assert L.pc_sts_count(_lib.RKG2, dt, dtE, 0) == osch.rkg2_iteration_count(dt, dtE)


@pytest.mark.parametrize("kind,s", [("rkl2", 2), ("rkl2", 45), ("rkl2", 447), ("rkg2", 3), ("rkg2", 55),
                                    ("rkg2", 547)])
def test_sts_tables_bitwise(L, kind, s):
    dt = 0.37
    out = np.zeros(5 * s)
    code = _lib.RKL2 if kind == "rkl2" else _lib.RKG2
    assert L.pc_sts_table(code, s, dt, _lib.dptr(out)) == 0
    ref = np.array(osch.stage_table(kind, s, dt))
    assert np.array_equal(out.reshape(s, 5), ref)
    assert not np.any(np.isnan(out))
