"""Diagnostic: stage-1 outputs of the uniform path on x-only smooth states,
saved for an offline search of the operation that differs from the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2210_06437_b200 import hydro  # noqa: E402

DX = 1.0 / 32
AX = int(os.environ.get("AXIS", "0"))
m = hydro.uniform_mesh(*[4 if k == AX else 1 for k in range(3)])
i = np.arange(512)
loc = (i & 7, (i >> 3) & 7, i >> 6)[AX]
x = ((m.pos[:, AX:AX + 1] * 8 + loc[None]) + 0.5) * DX  # [4, 512]
out = {}
cases = {
    "p_bump_vall": (1.0 + 0 * x, 0.1 + np.exp(-((x - 0.5) / 0.08) ** 2), (0.3, -0.1, 0.2)),
    "p_bump_vx": (1.0 + 0 * x, 0.1 + np.exp(-((x - 0.5) / 0.08) ** 2), (0.3, 0.0, 0.0)),
    "p_bump_v0": (1.0 + 0 * x, 0.1 + np.exp(-((x - 0.5) / 0.08) ** 2), (0.0, 0.0, 0.0)),
    "rho_p_bump_vx": (1.0 + 0.5 * np.exp(-((x - 0.5) / 0.08) ** 2), 0.1 + np.exp(-((x - 0.5) / 0.08) ** 2),
                      (0.3, 0.0, 0.0)),
    "p_bump_vy": (1.0 + 0 * x, 0.1 + np.exp(-((x - 0.5) / 0.08) ** 2), (0.0, -0.1, 0.0)),
}
for name, (rho, p, v) in cases.items():
    U0 = np.zeros((4, 6, 512))
    U0[:, 0] = rho
    for k in range(3):
        U0[:, 1 + k] = rho * v[k]
    eint = p / 0.4
    U0[:, 4] = eint + 0.5 * rho * (v[0] ** 2 + v[1] ** 2 + v[2] ** 2)
    U0[:, 5] = eint ** (1 / 1.4)
    d = hydro.CudaDevice(hydro.HydroConfig(dx=DX))
    d.set_mesh(m)
    d.upload(U0)
    dt = d.compute_dt()
    d.launch_stage(1, list(range(4)))
    d.synchronize()
    g1 = d.download_buffer(1)
    d.close()
    pr = oracle.params(nf=6, dx=DX)
    w1 = oracle.stage(pr, m.neighbor_ids, U0, U0, 1, dt / DX)
    nd = int((g1 != w1).sum())
    print("axis", AX, name, "dt", dt, "cells differing", nd, "max", float(np.abs(g1 - w1).max()))
    out[name + "_U0"] = U0
    out[name + "_gpu"] = g1
    out[name + "_orc"] = w1
    out[name + "_dt"] = np.array([dt])
np.savez(f"gpurun_out/parity_1d_ax{AX}.npz", **out)
