"""Multi-GPU parity check (run under torchrun, one rank per GPU):

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29511 tools/multigpu_check.py [--dims 4 4 8] [--steps 3] [--species 0]

Every rank steps its Morton chunk of the global mesh with cross-GPU halos
over NCCL (pack -> grouped send/recv -> unpack, interior sub-grids overlapped
with the exchange) and the dt max-allreduce; rank 0 then steps the whole mesh
alone on its GPU and every rank compares its sub-grids BITWISE against that.
Prints "MULTIGPU OK ..." on success, exits 1 otherwise.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2210_06437_b200 import hydro as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", type=int, nargs=3, default=[4, 4, 8])
    ap.add_argument("--periodic", default="")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--species", type=int, default=0)
    ap.add_argument("--recon", default="ppm")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "p2p-ce", "nccl"])
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 (two processes sharing one GPU through CUDA IPC, time-sliced): "
                         "the cross-rank path on a one-GPU box")
    ap.add_argument("--amr", default="", choices=["", "lshape", "ref4"],
                    help="multi-rank coarse-fine AMR: an L-shaped refinement of a 4^3 box, or the reference's own "
                         "levels-4 build_mesh octree (tests/golden), dealt along the Morton curve")
    ap.add_argument("--dropin", default="", choices=["", "stage", "grid"],
                    help="per-sub-grid drop-in steps (ts_hydro_launch_stage) between batched ones: every "
                         "sub-grid's launch on a rotating stream, scrambled, stage by stage (stage) or "
                         "sub-grid by sub-grid (grid: the host parks what is not ready)")
    ap.add_argument("--gravity", action="store_true",
                    help="self-gravity across the ranks (FMM over the global tree, densities all-gathered over "
                         "NCCL): a solve and two hydro + gravity steps, against one rank")
    ap.add_argument("--mismatch", action="store_true",
                    help="rank 1 makes one stepping call too many: it must fail with TS_ECOMM, not hang")
    a = ap.parse_args()
    if a.transport == "p2p-ce":  # P2P with copy-engine halos instead of the in-kernel push
        os.environ["TS_HYDRO_HALO"] = "ce"
    if a.mismatch:
        os.environ["TS_HYDRO_WAIT_TIMEOUT_MS"] = "2000"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = 0 if a.same_device else int(os.environ.get("LOCAL_RANK", rank))
    if a.same_device and a.transport == "nccl":
        raise SystemExit("NCCL refuses two ranks on one GPU: --same-device takes p2p / p2p-ce")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if a.amr:
        return amr_check(a, rank, world, local)
    cfg = H.HydroConfig(device_id=local, n_species=a.species, dx=1.0 / (8 * a.dims[0]), recon=a.recon)
    mesh = H.uniform_mesh(*a.dims, periodic=a.periodic, world=world)
    dev = H.CudaDevice(cfg)
    dev.set_mesh(mesh, rank)
    if a.transport == "nccl":
        uid = [H.CudaDevice.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        dev.comm_init(uid[0], world, rank)
    else:
        blobs = [None] * world
        dist.all_gather_object(blobs, dev.p2p_export())
        dev.p2p_import(blobs)
        if a.gravity:  # the gravity gather runs over NCCL next to the P2P halos
            uid = [H.CudaDevice.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            dev.comm_init(uid[0], world, rank)
    dev.init_random(2210)
    if a.gravity:
        return gravity_check(a, dev, cfg, rank, world)
    owned = dev.owned_ids()
    n_owned, n_proxy, n_interior = dev.local_counts()
    if a.mismatch:
        dev.step(1)
        dev.synchronize()
        code = 0
        if rank == 1:
            try:
                dev.step(1)
                dev.synchronize()
            except H.TsError as e:
                code = e.code
        dist.barrier()
        res = torch.tensor([code if rank == 1 else H.TS_ECOMM])
        dist.all_reduce(res, op=dist.ReduceOp.MIN)
        if rank == 0:
            print("MISMATCH DETECTED" if res.item() == H.TS_ECOMM else f"MISMATCH NOT DETECTED ({res.item()})",
                  flush=True)
        dist.destroy_process_group()
        return 0 if res.item() == H.TS_ECOMM else 1
    if a.dropin:
        # a batched step, then drop-in steps (the first takes the batched
        # stage 3's pushes; the next ones each other's), then a batched one
        dev.step(1)
        n = n_owned
        for step in range(max(a.steps - 2, 1)):
            perm = [(k * 37 + step * 11 + 5) % n for k in range(n)] if n % 37 else list(range(n))[::-1]
            order = ([(st, g) for st in (1, 2, 3) for g in perm] if a.dropin == "stage"
                     else [(st, g) for g in perm for st in (1, 2, 3)])
            for i, (st, g) in enumerate(order):
                dev.launch_stage(st, [g], stream_id=1 + i % 12, guid=g)
            dev.finish_step()
        dev.step(1)
        a.steps = max(a.steps - 2, 1) + 2
    else:
        # two calls: the first stage of each call refreshes the halos by a copy, the
        # other stages take the slabs the peers' stage kernels pushed
        dev.step(1)
        if a.steps > 1:
            dev.step(a.steps - 1)
    got = dev.download()
    dt = dev.last_dt()
    recs = [r for r in dev.flush_activity() if r.kind == "kernel"]
    launches = dev.launch_count()
    dev.close()

    # reference: the whole mesh on one GPU (each rank recomputes it on its own GPU)
    single = H.uniform_mesh(*a.dims, periodic=a.periodic, world=1)
    ref = H.CudaDevice(cfg)
    ref.set_mesh(single, 0)
    ref.init_random(2210)
    ref.step(a.steps)
    want = ref.download()[owned]
    dt_ref = ref.last_dt()
    ref.close()

    ok = bool(np.array_equal(got, want)) and dt == dt_ref
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    names = sorted({r.name for r in recs})
    print(f"rank {rank}: owned {n_owned} proxies {n_proxy} interior {n_interior} bitwise={ok} dt={dt!r} "
          f"launches={launches} kernels={names}", flush=True)
    dist.barrier()
    if rank == 0:
        print(("MULTIGPU OK" if flag.item() == 1 else "MULTIGPU FAIL") +
              f" world={world} dims={a.dims} steps={a.steps} species={a.species} transport={a.transport}"
              + (" same-device" if a.same_device else "") + (f" dropin={a.dropin}" if a.dropin else ""), flush=True)
    dist.destroy_process_group()
    return 0 if flag.item() == 1 else 1


def gravity_check(a, dev, cfg, rank, world):
    """Self-gravity on N ranks: one FMM solve of the random state, then two
    hydro + gravity steps; each rank's sub-grids bitwise equal to one rank."""
    owned = dev.owned_ids()
    dev.set_gravity_tree()
    dev.gravity_fmm(G=1.0, radius=2)
    g = dev.download_gravity()
    dev.step_gravity(2, G=1.0, radius=2)
    got = dev.download()
    dt = dev.last_dt()
    names = sorted({r.name for r in dev.flush_activity() if r.kind == "kernel"})
    dev.close()
    single = H.uniform_mesh(*a.dims, periodic=a.periodic, world=1)
    ref = H.CudaDevice(cfg)
    ref.set_mesh(single, 0)
    ref.init_random(2210)
    ref.set_gravity_tree()
    ref.gravity_fmm(G=1.0, radius=2)
    g_ref = ref.download_gravity()[owned]
    ref.step_gravity(2, G=1.0, radius=2)
    want = ref.download()[owned]
    dt_ref = ref.last_dt()
    ref.close()
    ok = bool(np.array_equal(g, g_ref)) and bool(np.array_equal(got, want)) and dt == dt_ref
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    print(f"rank {rank}: gravity bitwise={np.array_equal(g, g_ref)} steps bitwise={np.array_equal(got, want)} "
          f"dt={dt!r} kernels={names}", flush=True)
    dist.barrier()
    if rank == 0:
        print(("MULTIGPU OK" if flag.item() == 1 else "MULTIGPU FAIL") +
              f" gravity world={world} dims={a.dims} transport={a.transport}", flush=True)
    dist.destroy_process_group()
    return 0 if flag.item() == 1 else 1


def amr_check(a, rank, world, local):
    """Multi-rank AMR: each rank steps its Morton chunk of the leaves (ghost
    leaves refreshed whole before every stage, dt reduced over the ranks) and
    compares its leaves bitwise with the one-rank AMR run on its own GPU."""
    import json
    from paper_2210_06437_b200 import amr
    if a.amr == "lshape":
        mesh = amr.amr_mesh(4, 4, 4, {(0, 1, 1, 1), (0, 2, 1, 1), (0, 1, 2, 1), (0, 1, 1, 2), (0, 2, 2, 2)})
        dx, centre = 1.0 / 64, (0.625, 0.625, 0.5)
    else:
        vec = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_vectors.json")))
        m = max(vec["build_mesh"], key=lambda e: len(e["level"]))
        mesh = amr.from_reference_mesh(m["level"], m["pos"])
        dx, centre = 1.0 / (8 << mesh.max_level), (0.4, 0.55, 0.5)
    nf = 6 + a.species
    U0 = amr.ic_blast(mesh, nf, dx, width=0.08, centre=centre, drift=(0.3, -0.1, 0.2))
    owner = amr.partition(mesh, world)
    cfg = H.HydroConfig(device_id=local, n_species=a.species, dx=dx, recon=a.recon)
    dev = H.CudaDevice(cfg)
    dev.set_amr_mesh(mesh, owner=owner, rank=rank, world=world)
    if a.transport == "nccl":
        uid = [H.CudaDevice.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        dev.comm_init(uid[0], world, rank)
    else:
        blobs = [None] * world
        dist.all_gather_object(blobs, dev.p2p_export())
        dev.p2p_import(blobs)
    owned = dev.owned_ids()
    dev.upload(U0[owned])
    dev.step(1)
    if a.steps > 1:
        dev.step(a.steps - 1)
    got = dev.download()
    dt = dev.last_dt()
    n_owned, n_extra, _ = dev.local_counts()
    dev.close()
    ref = H.CudaDevice(cfg)
    ref.set_amr_mesh(mesh)
    ref.upload(U0[:mesh.n_leaves])
    ref.step(a.steps)
    want = ref.download()[owned]
    dt_ref = ref.last_dt()
    ref.close()
    ok = bool(np.array_equal(got, want)) and dt == dt_ref
    flag = torch.tensor([1 if ok else 0])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    print(f"rank {rank}: owned leaves {n_owned} ghost leaves + proxies {n_extra} bitwise={ok} dt={dt!r}", flush=True)
    dist.barrier()
    if rank == 0:
        print(("MULTIGPU OK" if flag.item() == 1 else "MULTIGPU FAIL") +
              f" AMR {a.amr} world={world} leaves={mesh.n_leaves} steps={a.steps} species={a.species} "
              f"transport={a.transport}" + (" same-device" if a.same_device else ""), flush=True)
    dist.destroy_process_group()
    return 0 if flag.item() == 1 else 1


if __name__ == "__main__":
    sys.exit(main())
