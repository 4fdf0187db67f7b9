"""cProfile of bench.py's C5 e2e leg (one untimed + one timed step): where the
host-side seconds above the device step go."""
import cProfile
import pstats
import sys
import types

sys.argv = ["bench.py"]
import bench  # noqa: E402
from paper_2403_01004_b200 import device, ptl  # noqa: E402

ctx = device.Context(0, 1, 0, None)
device.set_default_context(ctx)
prob = bench.Problem("c5", ctx)
args = types.SimpleNamespace(steps=1, warmup=1, pc="jacobi", scheme=None)
sc = bench.scheme_for("c5", args)
pr = cProfile.Profile()
pr.enable()
e = bench.run_e2e(args, prob, sc, ptl.PtlConfig(), ctx, None)
pr.disable()
print(e)
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(18)
