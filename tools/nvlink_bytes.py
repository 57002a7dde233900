"""NVLink bytes of the fused halo push against the halo plan (run under
torchrun, one rank per GPU):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29517 tools/nvlink_bytes.py [--steps 20] [--transport p2p|p2p-ce]

Each rank steps its Morton chunk of the weak-scaled Sedov mesh (16^3
sub-grids per GPU); around the timed steps it reads the NVML NVLink data
counters of its GPU (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, KiB, summed over
links) and compares the bytes per step with what the halo plan says must move:
per stage every slab a rank owes a peer (192 cells x nf x 8 B) plus the
rank's dt value.  Prints one JSON line per rank."""
import argparse
import json
import os
import sys

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2210_06437_b200 import hydro as H  # noqa: E402


def nvlink_kib(handle):
    import pynvml
    vals = []
    for fid in (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX):
        tot = 0
        for link in range(18):
            try:
                r = pynvml.nvmlDeviceGetFieldValues(handle, [(fid, link)])[0]
                if r.nvmlReturn == 0:
                    tot += r.value.ullVal
            except Exception:
                pass
        vals.append(tot)
    return vals


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--edge", type=int, default=16)
    ap.add_argument("--transport", default="p2p", choices=["p2p", "p2p-ce"])
    a = ap.parse_args()
    if a.transport == "p2p-ce":
        os.environ["TS_HYDRO_HALO"] = "ce"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import pynvml
    pynvml.nvmlInit()
    handle = pynvml.nvmlDeviceGetHandleByIndex(local)
    dims = (a.edge, a.edge, a.edge * world)
    cfg = H.HydroConfig(device_id=local, dx=1.0 / (8 * a.edge))
    mesh = H.uniform_mesh(*dims, world=world)
    dev = H.CudaDevice(cfg)
    session = H.WorkloadSession(mesh, dev, H.StepConfig(num_steps=a.steps), rank=rank)
    blobs = [None] * world
    dist.all_gather_object(blobs, dev.p2p_export())
    dev.p2p_import(blobs)
    session.load_problem("sedov")
    dev.compute_dt()
    dev.step(3)
    dev.synchronize()
    n_send = sum(len(dev.halo_plan(q)[0]) for q in range(world) if q != rank)
    slab_bytes = 192 * cfg.nf * 8
    plan = 3 * n_send * slab_bytes + 8 * (world - 1)  # per step: 3 stages of slabs + the dt value
    dist.barrier()
    before = nvlink_kib(handle)
    dev.step(a.steps)
    dev.synchronize()
    dist.barrier()
    after = nvlink_kib(handle)
    tx = (after[0] - before[0]) * 1024 / a.steps
    rx = (after[1] - before[1]) * 1024 / a.steps
    line = {"rank": rank, "world": world, "transport": a.transport, "steps": a.steps, "slabs_sent_per_stage": n_send,
            "plan_bytes_per_step": plan, "nvlink_tx_bytes_per_step": tx, "nvlink_rx_bytes_per_step": rx,
            "tx_over_plan": tx / plan if plan else None}
    print(json.dumps(line), flush=True)
    dev.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
