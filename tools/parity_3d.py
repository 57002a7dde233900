"""Diagnostic: stage-by-stage outputs of the uniform path (per-sub-grid
launches and the batched step) on a 3-D smooth bump with drift, saved for an
offline search of the operation that differs from the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2210_06437_b200 import amr, hydro  # noqa: E402

DX = 1.0 / 64
m0 = amr.amr_mesh(4, 4, 4, set())
m = hydro.uniform_mesh(4, 4, 4)
out = {}
for name, drift in (("drift", (0.3, -0.1, 0.2)), ("nodrift", (0.0, 0.0, 0.0))):
    U0 = amr.ic_blast(m0, 6, DX, width=0.06, centre=(0.3, 0.3, 0.25), drift=drift)
    pr = oracle.params(nf=6, dx=DX)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=DX))
    d.set_mesh(m)
    d.upload(U0)
    dt = d.compute_dt()
    every = list(range(m.n))
    g = []
    for k in (1, 2, 3):
        d.launch_stage(k, every)
        d.synchronize()
        g.append(d.download_buffer(k % 3))
    d.close()
    w1 = oracle.stage(pr, m.neighbor_ids, U0, U0, 1, dt / DX)
    w2 = oracle.stage(pr, m.neighbor_ids, g[0], U0, 2, dt / DX)
    w3 = oracle.stage(pr, m.neighbor_ids, g[1], U0, 3, dt / DX)
    for k, (a, b) in enumerate(zip(g, (w1, w2, w3)), 1):
        print(name, "stage", k, "(from the GPU's previous stage) cells differing", int((a != b).sum()),
              "max", float(np.abs(a - b).max()))
    out[name + "_U0"] = U0
    for k in range(3):
        out[f"{name}_gpu{k + 1}"] = g[k]
    out[name + "_dt"] = np.array([dt])
np.savez("gpurun_out/parity_3d.npz", **out)
