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
ts = []
for it in range(calls):
    ctx.sync()
    ctx.mark(0)
    prob.step(sc, ptl.PtlConfig())
    ctx.mark(1)
    ts.append(ctx.elapsed_ms(0, 1))
print(name, " ".join("%.1f" % t for t in ts), flush=True)
