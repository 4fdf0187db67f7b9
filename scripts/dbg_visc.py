import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
from helpers import oracle_geometry, soa, window_geometry
from oracle import ptl as optl
from paper_2403_01004_b200 import configs, device, operators
ctx = device.default_context()
n = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (768, 768, 1536)
w = configs.c5(n=n)
dg = device.device_grid(w.grid, w.bc, ctx)
rho = configs.gen_radial(device.DeviceField(dg, 1), w.meta["rho_r"])
v = configs.gen_harmonic(device.DeviceField(dg, 3), w.grid, w.seed)
cfg = operators.ScalarDiffusionConfig(nu=1.0, rho=rho, bc=w.bc, vector_metric=True)
op = operators.DiffusionOperator.scalar(cfg, 3)
dop = op.device_op(w.grid, 3, ctx)
F = device.DeviceField(dg, 3); F2 = device.DeviceField(dg, 3)
dop.apply(v, F); dop.apply(v, F2)
geom = oracle_geometry(w.grid, w.bc)
n0 = dg.shape[0]
for a in [1, n0 // 4, n0 // 2, n0 // 2 + 7, 3 * n0 // 4]:
    b = a + 3
    lo, hi = a - 1, b + 1
    gw = window_geometry(geom, lo, hi)
    r3 = w.meta["rho_r"][lo:hi, None, None] * np.ones((hi - lo,) + tuple(dg.shape[1:]))
    oop = optl.OracleOperator(gw, "scalar", 3, np.full(r3.shape, 1.0) * r3, r3, True)
    vw = soa(configs.harmonic_velocity(w.grid, w.seed, i0=lo, n0=hi - lo))
    vg = v.download_planes(lo, hi - lo)
    print("window", a, "input equal:", np.array_equal(vg, vw), flush=True)
    Fo = oop.apply(vw)[:, a - lo:b - lo]
    Fg = F.download_planes(a, 3); Fg2 = F2.download_planes(a, 3)
    bad = np.argwhere(Fg != Fo)
    print("  det:", np.array_equal(Fg, Fg2), "bad:", len(bad))
    if len(bad):
        for c in range(3):
            for p in range(3):
                bb = np.argwhere(Fg[c, p] != Fo[c, p])
                if len(bb):
                    print(f"   comp {c} plane {a+p}: {len(bb)} nodes j in {sorted(set(bb[:,0].tolist()))[:10]} k {bb[:,1].min()}..{bb[:,1].max()}")
