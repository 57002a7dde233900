"""Gravity slice throughput on the B200: near-field monopole P2P over the
Sedov 16^3 sub-grid mesh, radius 2/4/6; kernel time from the activity records
(device %globaltimer stamps); interactions/s and FP64 rate (4 DFMA = 8 flop per
interaction) against the FP64 peak (64 FMA lanes/SM/clk x 148 SMs x 1.965 GHz
= 37.2 TFLOP/s)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_06437_b200 import hydro as H  # noqa: E402
import oracle  # noqa: E402

m = H.uniform_mesh(16, 16, 16)
d = H.CudaDevice(H.HydroConfig(dx=1.0 / 128))
d.set_mesh(m)
d.upload(H.ic_fill(d.config, "sedov", m, np.arange(m.n)))
d.step(2)
peak = 148 * 64 * 2 * 1.965e9
for R in (2, 4, 6):
    n_st = len(oracle.p2p_stencil(R)[0])
    for _ in range(3):
        d.gravity_p2p(radius=R)
    d.synchronize()
    d.flush_activity()
    reps = 20
    for _ in range(reps):
        d.gravity_p2p(radius=R)
    d.synchronize()
    recs = [r for r in d.flush_activity() if r.name == "p2p_kernel"]
    t = np.median([r.end_ns - r.start_ns for r in recs]) * 1e-9
    inter = m.n * 512 * n_st
    print(json.dumps({"radius": R, "stencil": n_st, "sub_grids": m.n, "kernel_us": t * 1e6,
                      "interactions_per_s": inter / t, "fp64_tflops": 8 * inter / t / 1e12,
                      "fp64_frac_of_peak": 8 * inter / t / peak}), flush=True)
d.close()
