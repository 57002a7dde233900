"""Diagnostic: first step where the GPU AMR path and the oracle part on the
reference's golden octrees (per mesh, recon); prints the mismatching leaves
with their level and which faces point at proxies."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2210_06437_b200 import amr  # noqa: E402
from paper_2210_06437_b200 import hydro as H  # noqa: E402

vec = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_vectors.json")))
for m in vec["build_mesh"]:
    if m["levels"] < 3:
        continue
    a = amr.from_reference_mesh(m["level"], m["pos"])
    dx = 1.0 / (8 << a.max_level)
    for recon in (0, 1):
        U0 = amr.ic_blast(a, 6, dx, width=0.12, centre=(0.4, 0.55, 0.5), drift=(0.3, -0.1, 0.2))
        for steps in (1, 2, 4):
            ref, dts = oracle.run_amr(oracle.params(nf=6, recon=recon, dx=dx), a, U0, steps)
            d = H.CudaDevice(H.HydroConfig(dx=dx, recon=("ppm", "minmod")[recon]))
            d.set_amr_mesh(a)
            d.upload(U0[:a.n_leaves])
            d.step(steps)
            d.synchronize()
            U = d.download()
            dt = d.last_dt()
            d.close()
            bad = np.argwhere(U != ref[:a.n_leaves])
            print(f"levels={m['levels']} recon={recon} steps={steps}: dt {dt!r} vs {dts[-1]!r}; {len(bad)} values differ",
                  flush=True)
            if len(bad):
                leaves = sorted(set(int(g) for g in bad[:, 0]))
                for g in leaves[:8]:
                    px = [f for f in range(6) if a.nbr[g, f] >= a.n_leaves]
                    cells = bad[bad[:, 0] == g]
                    err = np.abs(U[g] - ref[g]).max()
                    print(f"   leaf {g} level {a.level[g]} pos {a.pos[g].tolist()} proxy faces {px} "
                          f"n={len(cells)} first cells {cells[:4, 1:].tolist()} maxerr {err:.3e}")
                break
