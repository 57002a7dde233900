"""Throughput of the coarse-fine AMR path next to the uniform
path on the same device: cell-updates/s (leaf cells x steps / device time,
CUDA events on the compute stream) and each kernel's share of GPU time from
the context's own activity records (ts_hydro_flush_activity).

    python tools/amr_bench.py [--base 16] [--refined 8] [--steps 20] [--species 0]

Mesh: a base^3 level-0 box whose central refined^3 level-0 positions are split
once (2:1 balanced by construction); smooth blast IC on the refined region.
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2210_06437_b200 import amr, hydro  # noqa: E402


def run(mesh, nf, species, steps, warmup, dx, uniform=None):
    d = hydro.CudaDevice(hydro.HydroConfig(dx=dx, n_species=species, activity_buffer_capacity=1 << 20))
    U0 = amr.ic_blast(mesh, nf, dx, width=0.15 * mesh.dims[0] * 8 * dx * 2 ** mesh.max_level / 4)
    if uniform is None:
        d.set_amr_mesh(mesh)
    else:
        d.set_mesh(uniform)
    d.upload(U0[:mesh.n_leaves])
    d.step(warmup)
    d.synchronize()
    d.flush_activity()
    ms = d.time_steps(steps)
    recs = d.flush_activity()
    d.close()
    by = collections.defaultdict(float)
    for r in recs:
        if r.kind == "kernel":
            by[r.name] += (r.end_ns - r.start_ns) * 1e-6
    tot = sum(by.values()) or 1.0
    return {"cell_updates_per_s": mesh.total_cells() * steps / (ms * 1e-3), "ms_per_step": ms / steps,
            "kernel_share": {k: round(v / tot, 4) for k, v in sorted(by.items())}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--base", type=int, default=16)
    ap.add_argument("--refined", type=int, default=8)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--species", type=int, default=0)
    a = ap.parse_args()
    lo = (a.base - a.refined) // 2
    mesh = amr.amr_mesh(a.base, a.base, a.base, lambda L, p: all(lo <= v < lo + a.refined for v in p))
    nf = 6 + a.species
    dx = 1.0 / (a.base * 16)
    out = {"workload": f"AMR {a.base}^3 level-0 box, central {a.refined}^3 refined once, nf {nf}",
           "leaves": mesh.n_leaves, "proxies": mesh.n_proxy, "reflux_records": len(mesh.reflux),
           "amr": run(mesh, nf, a.species, a.steps, a.warmup, dx)}
    # uniform reference point: the same number of leaves would not form a box,
    # so report the uniform base box at the finest dx (same kernel, no AMR work)
    um = amr.amr_mesh(a.base, a.base, a.base, set())
    out["uniform_base_box"] = run(um, nf, a.species, a.steps, a.warmup, dx / 2,
                                  uniform=hydro.uniform_mesh(a.base, a.base, a.base))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
