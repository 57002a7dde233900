"""Gravity FMM on the B200: one whole solve over the Sedov
16^3 sub-grid mesh (BASELINE config 2's mesh; 4681 octree nodes over 5
depths) and over an AMR mesh, radius 1/2/3.  Per-launch kernel times from the
activity records (device %globaltimer stamps), the solve's wall time on the
device from CUDA events around back-to-back solves, and the leaf pass's
interaction rate (4 DFMA per centred interaction) against the FP64 FMA peak
(64 lanes/SM/clk x 148 SMs x 1.965 GHz x 2 = 37.2 TFLOP/s)."""
import collections
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_06437_b200 import amr  # noqa: E402
from paper_2210_06437_b200 import hydro as H  # noqa: E402
import oracle  # noqa: E402

PEAK = 148 * 64 * 2 * 1.965e9


def run(name, d, leaves, reps=20):
    import torch
    for R in (1, 2, 3):
        for _ in range(3):
            d.gravity_fmm(radius=R)
        d.synchronize()
        d.flush_activity()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            d.gravity_fmm(radius=R)
        d.synchronize()
        e1.record()
        torch.cuda.synchronize()
        wall = e0.elapsed_time(e1) / reps * 1e-3
        per = collections.defaultdict(float)
        for r in d.flush_activity():
            if r.name.endswith("_kernel"):
                per[r.name] += (r.end_ns - r.start_ns) * 1e-9 / reps
        n_tab = len(oracle.fmm_table(R)[0])
        leaf_t = per.get("p2p_kernel", 0.0) + per.get("p2m_kernel", 0.0)
        inter = leaves * 512 * n_tab
        print(json.dumps({"mesh": name, "radius": R, "leaves": leaves, "solve_ms": wall * 1e3,
                          "kernel_ms": {k: round(v * 1e3, 4) for k, v in sorted(per.items())},
                          "leaf_interactions_per_s": inter / leaf_t if leaf_t else None,
                          "leaf_fp64_frac_of_peak": 8 * inter / leaf_t / PEAK if leaf_t else None}), flush=True)


def main():
    import torch
    torch.cuda.init()
    if "--ncu" in sys.argv:  # one solve per radius on the uniform mesh, for a profiler
        m = H.uniform_mesh(16, 16, 16, order="row")
        d = H.CudaDevice(H.HydroConfig(dx=1.0 / 128))
        d.set_mesh(m)
        d.upload(H.ic_fill(d.config, "sedov", m, np.arange(m.n)))
        d.set_gravity_tree()
        for R in (2, 3):
            d.gravity_fmm(radius=R)
        d.synchronize()
        d.close()
        return
    m = H.uniform_mesh(16, 16, 16, order="row")
    d = H.CudaDevice(H.HydroConfig(dx=1.0 / 128))
    d.set_mesh(m)
    d.upload(H.ic_fill(d.config, "sedov", m, np.arange(m.n)))
    d.step(2)
    d.set_gravity_tree()
    run("sedov 16^3 uniform", d, m.n)
    d.close()
    a = amr.amr_mesh(16, 16, 16, lambda L, p: all(6 <= v < 10 for v in p))
    dx = 1.0 / 256
    d = H.CudaDevice(H.HydroConfig(dx=dx))
    d.set_amr_mesh(a)
    d.upload(amr.ic_blast(a, 6, dx, width=0.2, centre=(1.0, 1.0, 1.0))[:a.n_leaves])
    d.set_gravity_tree()
    run("amr 16^3 + refined 4^3 centre", d, a.n_leaves)
    d.close()


def coupled():
    """Hydro with self-gravity (ts_hydro_step_gravity: step, FMM R = 2, kick)
    against the hydro step alone: the polytrope (config 3: 32^3 sub-grids,
    nf 11) and Sedov 16^3; device time per step from CUDA events around
    back-to-back calls."""
    import torch
    for name, dims, prob, species, dx in (("sedov 16^3", (16, 16, 16), "sedov", 0, 1.0 / 128),
                                          ("polytrope 32^3 nf 11", (32, 32, 32), "polytrope", 5, 1.0 / 256)):
        m = H.uniform_mesh(*dims, order="row")
        d = H.CudaDevice(H.HydroConfig(dx=dx, n_species=species))
        d.set_mesh(m)
        d.upload(H.ic_fill(d.config, prob, m, np.arange(m.n)))
        d.set_gravity_tree()
        out = {"mesh": name, "sub_grids": m.n}
        for what, fn in (("hydro_only", lambda: d.step(1)), ("hydro_plus_gravity", lambda: d.step_gravity(1, 1.0, 2))):
            for _ in range(3):
                fn()
            d.synchronize()
            reps = 10
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                fn()
            d.synchronize()
            e1.record()
            torch.cuda.synchronize()
            out[what + "_ms_per_step"] = e0.elapsed_time(e1) / reps
        out["gravity_share"] = 1 - out["hydro_only_ms_per_step"] / out["hydro_plus_gravity_ms_per_step"]
        d.close()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if "--coupled" in sys.argv:
        import torch
        torch.cuda.init()
        coupled()
    else:
        main()
