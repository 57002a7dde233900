"""The reference's scaling sweep (harness.cpp: measure_arm / run_scaling_sweep /
sweep_rows_from_times / write_sweep_csv) on B200s: one fixed mesh (strong
scaling, cells from the world-1 mesh as sweep_rows_from_times counts them),
each GPU count timed with the per-kernel timing hook on ("full": activity
stamps and records) and off ("disabled"), min over repetitions, max over ranks.

    python tools/harness_sweep.py                       # N = 1
    torchrun --nproc-per-node N ... tools/harness_sweep.py   # one JSON line per N
    python tools/harness_sweep.py --combine a.json b.json ... --csv out.csv

The combine step builds the rows with hydro.sweep_rows_from_times and writes
them with hydro.write_sweep_csv (the reference's CSV header, %.17g)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2210_06437_b200 import hydro as H  # noqa: E402

DIMS = (32, 32, 16)  # 16384 sub-grids, 8.4 M cells, fixed for every N


def measure(a):
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
    mesh = H.uniform_mesh(*DIMS, world=world, order="row")
    dev = H.CudaDevice(H.HydroConfig(device_id=local, dx=1.0 / (8 * DIMS[0]), activity_buffer_capacity=1 << 16))
    session = H.WorkloadSession(mesh, dev, H.StepConfig(num_steps=a.steps), rank=rank)
    if world > 1:
        blobs = [None] * world
        dist.all_gather_object(blobs, dev.p2p_export())
        dev.p2p_import(blobs)
    session.load_problem("sedov")
    dev.step(3)
    dev.synchronize()
    out = {}
    for arm, on in (("with", True), ("without", False)):
        if world > 1:
            dist.barrier()
        t = H.measure_arm(session, on, repetitions=a.reps)
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        out[arm] = t
    if rank == 0:
        print(json.dumps({"n": world, "time_with_s": out["with"], "time_without_s": out["without"],
                          "steps": a.steps, "total_cells": mesh.total_cells(), "mesh": list(DIMS)}), flush=True)
    dev.close()
    if world > 1:
        dist.destroy_process_group()


def combine(a):
    pts = []
    for f in a.combine:
        for line in open(f):
            if line.startswith("{"):
                pts.append(json.loads(line))
    pts.sort(key=lambda p: p["n"])
    rows = H.sweep_rows_from_times(pts[0]["total_cells"], pts[0]["steps"], [p["n"] for p in pts],
                                   [p["time_with_s"] for p in pts], [p["time_without_s"] for p in pts])
    with open(a.csv, "w") as f:
        H.write_sweep_csv(f, rows)
    for r in rows:
        print(json.dumps(r.__dict__))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--combine", nargs="*")
    ap.add_argument("--csv", default="sweep.csv")
    a = ap.parse_args()
    if a.combine:
        combine(a)
    else:
        measure(a)


if __name__ == "__main__":
    main()
