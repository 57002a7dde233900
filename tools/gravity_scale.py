"""Hydro + self-gravity across GPUs (config 4 with gravity un-frozen).

Run under torchrun, one rank per GPU:
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tools/gravity_scale.py [--dims 32 32 16] [--steps 5]

Weak scaling: each rank owns dims[0] x dims[1] x dims[2] sub-grids (the mesh
is dims[2] x N deep), the binary initial model (config 4's two polytropes, nf
11), Morton chunks.  Per step: the batched hydro step alone (ts_hydro_step)
and hydro + FMM (R = 2) + kick (ts_hydro_step_gravity).  Halos over the fused
P2P push, the gravity's density all-gather over NCCL.  Times: max over ranks
of the host-observed time of K synchronised steps (device work is
stream-ordered behind a barrier; this is a tool, bench.py carries the
contract's device-timed numbers)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2210_06437_b200 import hydro as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=3, default=[32, 32, 16])
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    dims = (a.dims[0], a.dims[1], a.dims[2] * world)
    mesh = H.uniform_mesh(*dims, world=world)
    cfg = H.HydroConfig(device_id=local, n_species=5, dx=1.0 / (8 * dims[0]))
    d = H.CudaDevice(cfg)
    d.set_mesh(mesh, rank)
    if world > 1:
        blobs = [None] * world
        dist.all_gather_object(blobs, d.p2p_export())
        d.p2p_import(blobs)
        uid = [H.CudaDevice.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        d.comm_init(uid[0], world, rank)
    owned = d.owned_ids()
    d.upload(H.ic_fill(cfg, "binary", mesh, owned))
    d.set_gravity_tree()
    out = {"n_gpus": world, "sub_grids_per_gpu": int(len(owned)), "mesh": list(dims)}
    for what, fn in (("hydro", lambda: d.step(1)), ("hydro_gravity", lambda: d.step_gravity(1, 1.0, 2))):
        for _ in range(2):
            fn()
        d.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            fn()
        d.synchronize()
        t = (time.perf_counter() - t0) / a.steps
        tt = torch.tensor([t])
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        out[what + "_ms_per_step"] = tt.item() * 1e3
    cells = len(owned) * 512 * world
    out["hydro_gravity_cell_updates_per_s"] = cells / (out["hydro_gravity_ms_per_step"] * 1e-3)
    out["gravity_share"] = 1 - out["hydro_ms_per_step"] / out["hydro_gravity_ms_per_step"]
    d.close()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
