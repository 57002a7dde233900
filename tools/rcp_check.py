"""Diagnostic (TS_HYDRO_LIB=<...>/libts_hydro_rcpchk.so): run the drifting-bump
parity state and print the operands where the branch-free reciprocal differed
from IEEE 1.0 / x inside the stage kernel."""
import ctypes
import os
import struct
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_06437_b200 import hydro  # noqa: E402

# a fresh process has fresh device globals: repeat one step here
from paper_2210_06437_b200 import amr  # noqa: E402
m0 = amr.amr_mesh(4, 4, 4, set())
U0 = amr.ic_blast(m0, 6, 1 / 64, width=0.06, centre=(0.3, 0.3, 0.25), drift=(0.3, -0.1, 0.2))
d = hydro.CudaDevice(hydro.HydroConfig(dx=1 / 64))
d.set_mesh(hydro.uniform_mesh(4, 4, 4))
d.upload(U0)
d.step(1)
d.synchronize()
L = hydro.lib()
L.ts_debug_rcp_bad.restype = ctypes.c_longlong
out = np.zeros((64, 3))
n = L.ts_debug_rcp_bad(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 64)
print("mismatching reciprocals:", n)
hx = lambda v: struct.unpack("<Q", struct.pack("<d", v))[0]
for x, y, z in out[:min(n, 20)]:
    print(f"x={x!r} ({hx(x):016x}) rcp_rn={y!r} ({hx(y):016x}) ieee={z!r} ({hx(z):016x})")
