"""Per-rank kernel timeline of a few steps from the library's own activity
records (in-kernel globaltimer stamps).  Single GPU or under torchrun:

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29512 tools/timeline.py [--edge 16] [--steps 2]
"""
import argparse
import os
import sys

import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2210_06437_b200 import hydro as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--edge", type=int, default=16)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--species", type=int, default=0)
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"])
    ap.add_argument("--quiet", action="store_true", help="totals and summary only")
    ap.add_argument("--replicas", action="store_true", help="every rank steps its own single-GPU mesh")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    rep = a.replicas and world > 1
    mesh = (H.uniform_mesh(a.edge, a.edge, a.edge) if rep else H.uniform_mesh(a.edge, a.edge, a.edge * world, world=world))
    dev = H.CudaDevice(H.HydroConfig(device_id=local, dx=1.0 / (8 * a.edge), n_species=a.species))
    dev.set_mesh(mesh, 0 if rep else rank)
    if rep:
        pass
    elif world > 1 and a.transport == "nccl":
        uid = [H.CudaDevice.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        dev.comm_init(uid[0], world, rank)
    elif world > 1:
        blobs = [None] * world
        dist.all_gather_object(blobs, dev.p2p_export())
        dev.p2p_import(blobs)
    dev.init_random(1)
    dev.step(10)
    dev.synchronize()
    dev.flush_activity()
    if world > 1:
        dist.barrier()
    ms = dev.time_steps(a.steps)
    recs = sorted((r for r in dev.flush_activity() if r.kind == "kernel"), key=lambda r: r.start_ns)
    t0 = recs[0].start_ns if recs else 0
    lines = [f"rank {rank}: {a.steps} steps in {ms:.3f} ms (event-timed); owned/proxy/interior {dev.local_counts()}"]
    busy = 0
    for r in recs:
        lines.append(f"  {r.name:22s} s{r.stream_id} {(r.start_ns - t0) / 1e3:9.1f} -> {(r.end_ns - t0) / 1e3:9.1f} us"
                     f"  ({(r.end_ns - r.start_ns) / 1e3:7.1f})")
    # per-kernel mean duration and the mean idle gap before each stage kernel
    from collections import defaultdict
    dur, gaps = defaultdict(list), []
    prev_end = None
    for r in recs:
        dur[r.name].append((r.end_ns - r.start_ns) / 1e3)
        if r.name.startswith("hydro_stage"):
            if prev_end is not None:
                gaps.append((r.start_ns - prev_end) / 1e3)
            prev_end = r.end_ns
    summ = "  summary: " + ", ".join(f"{k} {sum(v) / len(v):.1f} us x{len(v)}" for k, v in sorted(dur.items()))
    if gaps:
        summ += f", stage gap {sum(gaps) / len(gaps):.1f} us"
    lines.insert(1, summ)
    if a.quiet:
        lines = lines[:2]
    text = "\n".join(lines)
    if world > 1:
        out = [None] * world
        dist.all_gather_object(out, text)
        if rank == 0:
            print("\n".join(out))
        dist.destroy_process_group()
    else:
        print(text)


if __name__ == "__main__":
    main()
