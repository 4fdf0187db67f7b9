"""Probe the host<->device legs of the C5 e2e step: pinned H2D / D2H rates of
1- and 3-component fields through DeviceField.upload / download (the C-ABI
pc_field_upload / pc_field_download)."""
import time

import numpy as np

from paper_2403_01004_b200 import configs, device

w = configs.c5(host=False)
ctx = device.default_context()
dg = device.device_grid(w.grid, w.bc, ctx)
n = tuple(w.grid.shape)
for nc in (1, 3):
    a = device.pinned_empty(n + (nc,))
    a[...] = 1.0
    f = device.DeviceField(dg, nc)
    for rep in range(2):
        ctx.sync()
        t = time.perf_counter()
        f.upload(a)
        ctx.sync()
        tu = time.perf_counter() - t
        t = time.perf_counter()
        f.download(a)
        ctx.sync()
        td = time.perf_counter() - t
        print(f"ncomp {nc} rep {rep}: {a.nbytes/1e9:.2f} GB  H2D {a.nbytes/tu/1e9:.1f} GB/s ({tu:.3f} s)  "
              f"D2H {a.nbytes/td/1e9:.1f} GB/s ({td:.3f} s)", flush=True)
    b = np.empty_like(a)  # pageable target/source
    b[...] = 1.0
    t = time.perf_counter()
    f.upload(b)
    ctx.sync()
    tu = time.perf_counter() - t
    print(f"ncomp {nc} pageable H2D {b.nbytes/tu/1e9:.1f} GB/s", flush=True)
    del f, a, b
