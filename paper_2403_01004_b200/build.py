"""Build the sm_100a CUDA library in-tree (no JIT cache, travels with gpurun).

    python -m paper_2403_01004_b200.build

produces ``paper_2403_01004_b200/_lib/libparacycle_b200.so``.  Flags:
  -gencode arch=compute_100a,code=sm_100a   B200 only
  -fmad=false / -ffp-contract=off           bitwise parity with the numpy oracle
  -lineinfo                                 ncu source view
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libparacycle_b200.so")
SOURCES = ["capi.cu"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "-shared",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "paracycle_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    extra = os.environ.get("PC_NVCC_EXTRA", "").split()  # experiments only, e.g. -DSMARCH_MINB=2
    flags = NVCC_FLAGS
    if os.environ.get("PC_FMAD") == "1":  # experiment: contraction on (NOT bitwise with the oracle)
        flags = [f for f in flags if f != "-fmad=false"]
        flags = [f.replace(",-ffp-contract=off", "") for f in flags]
    cmd = [_nvcc(), *flags, *extra, "-o", LIB + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(OUT_DIR, "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stderr[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(LIB + ".tmp", LIB)
    if verbose:
        sys.stderr.write(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
