import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from paper_2403_01004_b200 import configs, operators, ptl, schemes, device
w = configs.c3(n=(20, 40, 64))
cfg = operators.AlignedConductionConfig(b_hat=w.fields["b"], m_p=3.0, k_B=1.0, bc=w.bc)
op = operators.DiffusionOperator.aligned(cfg, operators.Field(w.grid, w.fields["T"]))
dop = op.device_op(w.grid, 1)
print("dtE", dop.dt_euler, flush=True)
u = device.DeviceField.from_values(dop.dgrid, w.fields["T"])
F = device.DeviceField(dop.dgrid, 1)
dop.apply(u, F); dop.ctx.sync(); print("apply ok", flush=True)
from paper_2403_01004_b200 import _lib
import ctypes
L = _lib.lib()
p, lim, k = ctypes.c_double(), ctypes.c_int(), ctypes.c_int64()
_lib.check(L.pc_ptl(dop.dgrid.handle, u.handle, F.handle, 1e-12, 0, ctypes.byref(p), ctypes.byref(lim), ctypes.byref(k)))
print("ptl ok", p.value, lim.value, k.value, flush=True)
for s in (2, 3, 5):
    _lib.check(L.pc_step_sts(dop.handle, u.handle, 10 * dop.dt_euler, 0, s, None)); dop.ctx.sync()
    print("sts", s, "ok", flush=True)
out, rep = ptl.cycle_operator(op, schemes.SchemeConfig("rkl2"), operators.Field(w.grid, w.fields["T"]), 100 * dop.dt_euler)
print("cycle ok", rep.n_cycles, flush=True)
