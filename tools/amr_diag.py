"""Diagnostic: where does the GPU AMR path differ from the oracle after one
step?  Compares U^(1) (buffer B), U^(2) (C) and U^(n+1) (A) per stage."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2210_06437_b200 import amr, hydro  # noqa: E402

DX = 1.0 / 64
L_SHAPE = {(0, 1, 1, 1), (0, 2, 1, 1), (0, 1, 2, 1), (0, 1, 1, 2), (0, 2, 2, 2)}
drift = tuple(float(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (0.3, -0.1, 0.2)
m = amr.amr_mesh(4, 4, 4, L_SHAPE)
U0 = amr.ic_blast(m, 6, DX, width=0.06, centre=(0.625, 0.625, 0.5), drift=drift)
p = oracle.params(nf=6, dx=DX)
d = hydro.CudaDevice(hydro.HydroConfig(dx=DX))
d.set_amr_mesh(m)
d.upload(U0[:m.n_leaves])
d.step(1)
d.synchronize()
dt = d.last_dt()
G = {1: d.download_buffer(1), 2: d.download_buffer(2), 3: d.download_buffer(0)}
d.close()
amax = oracle.max_signal_speed(p, U0[:m.n_leaves])
dt_o = (p.cfl * p.dx) / amax
print("drift", drift, "dt gpu", dt, "oracle", dt_o, dt == dt_o)
U = U0.copy()
prev = U.copy()
for k in (1, 2, 3):
    for rf in (True, False):
        out = oracle.amr_stage(p, m, prev.copy(), U, k, dt_o, reflux=rf)
        diff = np.abs(G[k] - out[:m.n_leaves])
        bad = np.argwhere(diff > 0)
        print(f"stage {k} reflux={rf}: max diff {diff.max():.3e}, cells differing {len(bad)}")
        if rf and len(bad):
            for L in range(m.max_level + 1):
                sel = m.level[bad[:, 0]] == L
                print(f"   level {L}: {sel.sum()} cells, leaves {len(set(bad[sel, 0]))}")
            for g, f, c in bad[:8]:
                print("   leaf", g, "level", m.level[g], "field", f, "cell", (c & 7, (c >> 3) & 7, c >> 6),
                      "nbr", m.nbr[g].tolist(), "gpu", G[k][g, f, c], "orc", out[g, f, c])
        if rf:
            keep = out
    prev = np.zeros_like(U)
    prev[:m.n_leaves] = G[k]  # continue from the GPU's state to isolate each stage
