"""Stage-by-stage GPU vs oracle diagnostic: first mismatching cell per stage."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2210_06437_b200 import hydro as H  # noqa: E402

problem = sys.argv[1] if len(sys.argv) > 1 else "binary"
species = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dims = (4, 4, 2)
m = H.uniform_mesh(*dims)
cfg = H.HydroConfig(dx=1.0 / 32, n_species=species)
U0 = H.ic_fill(cfg, problem, m, np.arange(m.n))
p = oracle.params(nf=cfg.nf, dx=cfg.dx)
d = H.CudaDevice(cfg)
d.set_mesh(m)
d.upload(U0)
dt_gpu = d.compute_dt()
amax = oracle.max_signal_speed(p, U0)
dtdx = ((p.cfl * p.dx) / amax) / p.dx
print("dt gpu", dt_gpu, "oracle", (p.cfl * p.dx) / amax)
Uprev = U0
outs = []
for st in (1, 2, 3):
    d.synchronize()
    for g in range(m.n):
        d.launch_stage(st, [g])
    d.synchronize()
    got = d.download_buffer({1: 1, 2: 2, 3: 0}[st])
    want = oracle.stage(p, m.neighbor_ids, Uprev, U0, st, dtdx)
    bad = np.argwhere(got != want)
    print(f"stage {st}: {len(bad)} mismatching values")
    for g, f, c in bad[:8]:
        z, y, x = c // 64, (c // 8) % 8, c % 8
        print(f"  g={g} f={f} cell=({x},{y},{z}) gpu={got[g, f, c]!r} oracle={want[g, f, c]!r} diff={got[g, f, c] - want[g, f, c]:.3e}")
    if len(bad):
        g, f, c = bad[0]
        print("  Uprev fields at that cell:", [Uprev[g, k, c] for k in range(cfg.nf)])
        break
    Uprev = want
    if st == 3:
        break
d.close()
