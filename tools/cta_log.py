"""Per-CTA timeline of one step (TS_HYDRO_CTA_LOG): where a stage's time goes.
Single GPU or under torchrun (fused P2P halos).  Prints per stage: span,
CTA duration (work) and wait (start -> work start) for boundary vs interior
CTAs, and how late the last CTA of each kind finished."""
import os
import sys

os.environ["TS_HYDRO_CTA_LOG"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2210_06437_b200 import hydro as H  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
if world > 1:
    dist.init_process_group("gloo", rank=rank, world_size=world)
edge = 16
mesh = H.uniform_mesh(edge, edge, edge * world, world=world)
dev = H.CudaDevice(H.HydroConfig(device_id=local, dx=1.0 / (8 * edge)))
dev.set_mesh(mesh, rank)
if world > 1:
    blobs = [None] * world
    dist.all_gather_object(blobs, dev.p2p_export())
    dev.p2p_import(blobs)
dev.init_random(7)
dev.compute_dt()
dev.step(5)
dev.synchronize()
log = dev.debug_cta_log().astype(np.int64)
n_owned, n_proxy, n_int = dev.local_counts()
owned = dev.owned_ids()
is_b = np.zeros(n_owned, bool)
if world > 1:
    for g in range(n_owned):
        nb = mesh.neighbor_ids[owned[g]]
        is_b[g] = any(x >= 0 and mesh.owner[x] != rank for x in nb)
t0 = log[:, :, 1].min()
out = [f"rank {rank}: boundary CTAs {int(is_b.sum())}"]
for s in range(3):
    L = log[s]
    span = (L[:, 3].max() - L[:, 1].min()) / 1e3
    work = (L[:, 3] - L[:, 2]) / 1e3
    wait = (L[:, 2] - L[:, 1]) / 1e3
    # CTA launch position -> sub-grid: boundary CTAs are the first n_b positions in the fused order
    nb = int(is_b.sum())
    pos_b = np.arange(len(L)) < nb
    line = (f"  stage {s + 1}: span {span:7.1f} us  start {(L[:, 1].min() - t0) / 1e3:8.1f}  "
            f"work med {np.median(work):5.1f} (b {np.median(work[pos_b]) if nb else 0:5.1f})  "
            f"wait>1us {int((wait > 1).sum())} (b {int((wait[pos_b] > 1).sum()) if nb else 0}) max wait {wait.max():6.1f}  "
            f"last end b {((L[pos_b, 3].max() - L[:, 1].min()) / 1e3) if nb else 0:6.1f} / all {span:6.1f}")
    out.append(line)
print("\n".join(out), flush=True)
