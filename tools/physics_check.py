"""Physical validity of a run: min density / pressure and non-finite counts after k steps."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_06437_b200 import hydro as H  # noqa: E402

problem, species = sys.argv[1], int(sys.argv[2])
dims = tuple(int(x) for x in sys.argv[3].split("x"))
steps = [int(s) for s in sys.argv[4].split(",")]
m = H.uniform_mesh(*dims)
cfg = H.HydroConfig(dx=1.0 / (8 * dims[0]), n_species=species)
d = H.CudaDevice(cfg)
d.set_mesh(m)
d.upload(H.ic_fill(cfg, problem, m, np.arange(m.n)))
done = 0
for s in steps:
    d.step(s - done)
    done = s
    U = d.download()
    rho = U[:, 0]
    E = U[:, 4]
    ke = 0.5 * (U[:, 1] ** 2 + U[:, 2] ** 2 + U[:, 3] ** 2) / np.where(rho > 0, rho, np.nan)
    p = (cfg.gamma - 1) * (E - ke)
    print(f"{problem} {dims} step {s}: nonfinite {int((~np.isfinite(U)).sum())}, rho<=0 {int((rho <= 0).sum())}, "
          f"min rho {np.nanmin(rho):.3e}, p<=0 {int((p <= 0).sum())}, dt {d.last_dt():.3e}")
d.close()
