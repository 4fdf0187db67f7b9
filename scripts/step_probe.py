"""Per-call device time of bench steps inside one process (no clock sampler,
no timing spans): python scripts/step_probe.py c2 [calls]"""
import sys
import types

name = sys.argv[1]
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sys.argv = ["bench.py"]
import bench  # noqa: E402
from paper_2403_01004_b200 import device, ptl  # noqa: E402

ctx = device.Context(0, 1, 0, None)
device.set_default_context(ctx)
prob = bench.Problem(name, ctx)
sc = bench.scheme_for(name, types.SimpleNamespace(steps=1, warmup=1, pc="jacobi", scheme=None))
import os  # noqa: E402
if os.environ.get("PROBE_TIMING"):
    ctx.enable_timing(True)
ts = []
for it in range(calls):
    ctx.sync()
    ctx.mark(0)
    prob.step(sc, ptl.PtlConfig())
    ctx.mark(1)
    ts.append(ctx.elapsed_ms(0, 1))
print(name, " ".join("%.1f" % t for t in ts), flush=True)
if os.environ.get("PROBE_TIMING"):
    for k, d in ctx.stats_by_kind().items():
        if d["launches"]:
            print("  %-12s %8.2f ms  %6d launches  %.1f us/launch" % (k, d["ms"], d["launches"],
                                                                     1e3 * d["ms"] / d["launches"]))
