"""C1 persistent-loop timing per call inside one process (no clock sampler):
is the spread per call or per process?"""
import sys
import time

import numpy as np

sys.argv = ["bench.py"]
import bench  # noqa: E402
from paper_2403_01004_b200 import device, ptl  # noqa: E402

ctx = device.Context(0, 1, 0, None)
device.set_default_context(ctx)
prob = bench.Problem("c1", ctx)
import types  # noqa: E402
args = types.SimpleNamespace(steps=1, warmup=1, pc="jacobi", scheme=None)
sc = bench.scheme_for("c1", args)
ts = []
for it in range(15):
    ctx.sync()
    ctx.mark(0)
    prob.step(sc, ptl.PtlConfig())
    ctx.mark(1)
    ts.append(ctx.elapsed_ms(0, 1))
print(" ".join("%.1f" % t for t in ts), flush=True)
