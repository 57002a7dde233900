"""Diagnostic: the uniform (set_mesh) path on the drift + bump state."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2210_06437_b200 import amr, hydro  # noqa: E402

DX = 1.0 / 64
m0 = amr.amr_mesh(4, 4, 4, set())
for drift in ((0.3, -0.1, 0.2), (0.0, 0.0, 0.0), (0.25, -0.125, 0.5)):
    U0 = amr.ic_blast(m0, 6, DX, width=0.06, centre=(0.3, 0.3, 0.25), drift=drift)
    p = oracle.params(nf=6, dx=DX)
    nbr, pos, owner = oracle.uniform_mesh(4, 4, 4)
    ref, dts = oracle.run(p, nbr, U0, 1)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=DX))
    d.set_mesh(hydro.uniform_mesh(4, 4, 4))
    d.upload(U0)
    d.step(1)
    d.synchronize()
    U = d.download()
    d.close()
    diff = np.abs(U - ref)
    bad = np.argwhere(diff > 0)
    print(os.environ.get("TS_HYDRO_FLOW", "flow default"), drift, f"max diff {diff.max():.3e} cells {len(bad)}")
    for g, f, c in bad[:6]:
        print("   ", g, f, (c & 7, (c >> 3) & 7, c >> 6), repr(U[g, f, c]), repr(ref[g, f, c]), repr(U0[g, f, c]))
