import mmap, time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2403_01004_b200 import configs, device
ctx = device.default_context()
w = configs.c5(n=(384, 768, 1536))
dg = device.device_grid(w.grid, w.bc, ctx)
f = configs.gen_temperature(device.DeviceField(dg, 1), w.grid, w.seed)
nbytes = dg.ncells * 8
def t(label, fn):
    t0 = time.perf_counter(); r = fn(); print(f"{label:40s} {time.perf_counter() - t0:7.3f} s  ({nbytes / 1e9:.2f} GB)", flush=True); return r
t("download into fresh np.empty", lambda: f.download())
a = np.empty(dg.shape + (1,)); a.fill(0.0)
t("download into pre-touched array", lambda: f.download(a))
def huge():
    m = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    m.madvise(mmap.MADV_HUGEPAGE)
    b = np.frombuffer(m, dtype=np.float64).reshape(dg.shape + (1,))
    f.download(b)
    return b
t("download into fresh MADV_HUGEPAGE mmap", huge)
ctx.pin(a)
t("download into registered (pinned) array", lambda: f.download(a))
t("pin (cudaHostRegister) a fresh array", lambda: ctx.pin(np.empty(dg.shape + (1,))))
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read())
