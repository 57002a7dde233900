"""BASELINE config 5: sub-grid batch sweep (fused-kernel throughput vs batch
size).  Single GPU, or under torchrun for the halo-overlap sweep (sizes are
per GPU, weak scaling along z).

    python tools/sweep.py [--species 0 5] [--sizes 256 1024 4096 16384 65536 262144] [--steps 10]

Prints one JSON line per (nf, size): cell-updates/s (max-over-ranks device
time), HBM roofline fraction of the measured copy bandwidth, stage-kernel time
share, and — at N > 1 — the halo pack/unpack time and how much of the step the
boundary launches add over the interior ones.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2210_06437_b200 import hydro as H  # noqa: E402

SHAPES = {256: (8, 8, 4), 1024: (16, 8, 8), 4096: (16, 16, 16), 16384: (32, 32, 16), 65536: (64, 32, 32),
          262144: (64, 64, 64)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--species", type=int, nargs="+", default=[0, 5])
    ap.add_argument("--sizes", type=int, nargs="+", default=sorted(SHAPES))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--recon", default="ppm")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"])
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = json.load(f)["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    for species in a.species:
        nf = 6 + species
        for n in a.sizes:
            nx, ny, nz = SHAPES[n]
            mesh = H.uniform_mesh(nx, ny, nz * world, world=world)
            dev = H.CudaDevice(H.HydroConfig(device_id=local, n_species=species, dx=1.0 / (8 * nx),
                                             recon=a.recon))
            dev.set_mesh(mesh, rank)
            if world > 1 and a.transport == "nccl":
                uid = [H.CudaDevice.nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(uid, src=0)
                dev.comm_init(uid[0], world, rank)
            elif world > 1:  # the default fused P2P halo push (bench.py's transport)
                blobs = [None] * world
                dist.all_gather_object(blobs, dev.p2p_export())
                dev.p2p_import(blobs)
            dev.init_random(2210)
            dev.step(3)
            dev.synchronize()
            dev.flush_activity()
            if world > 1:
                dist.barrier()
            ms = dev.time_steps(a.steps)
            recs = [r for r in dev.flush_activity() if r.kind == "kernel"]
            if world > 1:
                import torch
                t = torch.tensor([ms], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            stage_ns = sum(r.end_ns - r.start_ns for r in recs if r.name.startswith("hydro_stage"))
            halo_ns = sum(r.end_ns - r.start_ns for r in recs if r.name.startswith("halo_"))
            cells = mesh.n * 512
            value = cells * a.steps / (ms * 1e-3)
            per_gpu = value / world
            line = {"nf": nf, "subgrids_per_gpu": n, "gpus": world, "recon": a.recon,
                    "transport": a.transport if world > 1 else None,
                    "cell_updates_per_s": value, "ms_per_step": ms / a.steps,
                    "hbm_frac": per_gpu * 64 * nf / (hbm * 1e9),
                    "stage_kernel_share": stage_ns * 1e-6 / ms, "halo_kernels_ms_per_step": halo_ns * 1e-6 / a.steps}
            if rank == 0:
                print(json.dumps(line), flush=True)
            dev.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
