"""Diagnostic: isolate the stage kernel's per-level dx (a), the AMR path
without the flux correction (b) and with it (c), one step each."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2210_06437_b200 import amr, hydro  # noqa: E402

DX = 1.0 / 64
L_SHAPE = {(0, 1, 1, 1), (0, 2, 1, 1), (0, 1, 2, 1), (0, 1, 1, 2), (0, 2, 2, 2)}


def compare(tag, m, U0, steps=1):
    p = oracle.params(nf=6, dx=DX)
    ref, dts = oracle.run_amr(p, m, U0, steps)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=DX))
    d.set_amr_mesh(m)
    d.upload(U0[:m.n_leaves])
    d.step(steps)
    d.synchronize()
    U = d.download()
    dt = d.last_dt()
    d.close()
    diff = np.abs(U - ref[:m.n_leaves])
    bad = np.argwhere(diff > 0)
    print(f"{tag}: dt equal {dt == dts[-1]}, max diff {diff.max():.3e}, cells {len(bad)}, leaves "
          f"{sorted(set(bad[:, 0].tolist()))[:20]}")


U_drift = lambda m: amr.ic_blast(m, 6, DX, width=0.06, centre=(0.625, 0.625, 0.5), drift=(0.3, -0.1, 0.2))
m0 = amr.amr_mesh(4, 4, 4, set())
compare("(a0) uniform via AMR, max_level 0", m0, amr.ic_blast(m0, 6, DX, width=0.06, centre=(0.3, 0.3, 0.25),
                                                               drift=(0.3, -0.1, 0.2)))
mf = amr.AmrMesh(m0.dims, 1, m0.level, m0.pos, m0.nbr, np.array([0, 64, 64]), m0.proxies, m0.reflux)
compare("(a1) level-0 leaves, dx_upd = 2 dx", mf, amr.ic_blast(m0, 6, DX, width=0.06, centre=(0.3, 0.3, 0.25),
                                                                drift=(0.3, -0.1, 0.2)))
m = amr.amr_mesh(4, 4, 4, L_SHAPE)
mb = amr.AmrMesh(m.dims, m.max_level, m.level, m.pos, m.nbr, m.level_first, m.proxies, m.reflux[:0])
compare("(b) L-shape, no reflux", mb, U_drift(m))
compare("(c) L-shape", m, U_drift(m))
compare("(c0) L-shape, no drift", m, amr.ic_blast(m, 6, DX, width=0.06, centre=(0.625, 0.625, 0.5)))
compare("(c3) L-shape, 3 steps", m, U_drift(m), 3)
