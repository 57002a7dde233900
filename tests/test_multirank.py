"""N>1 host logic on CPU (gloo, world size 2): the library's halo plans and
the packed-slab wire format drive a partitioned oracle step whose result must
be bitwise equal to the single-domain step — the multi-GPU analogue of the
reference's comm-mode equivalence (test_workload.cpp:317-331, 448-464).

Each rank: host-only context (device_id = -1) -> owned sub-grids, proxies and
per-peer plans; packs the 3-deep slabs it owes each peer into ONE message per
directed rank pair (the aggregated exchange), exchanges over gloo, unpacks
into its proxies, runs the three SSP-RK3 stages on its own sub-grids with the
dt max-allreduce between steps."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.conftest import ROOT

N = 8


def slab_cells(face):
    """Slab cell offsets of `face` in wire order k = l + 3 (u + 8 v) (hydro_kernels.cu slab_cell)."""
    axis = face // 2
    out = []
    for v in range(N):
        for u in range(N):
            for l in range(3):
                d = N - 3 + l if face & 1 else l
                x, y, z = [(d, u, v), (u, d, v), (u, v, d)][axis]
                out.append((z * N + y) * N + x)
    return np.array(out, np.int64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, dims, periodic, steps, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2210_06437_b200 import hydro as H
    try:
        mesh = H.uniform_mesh(*dims, periodic=periodic, world=world)
        dev = H.CudaDevice(H.HydroConfig(device_id=-1, n_species=1))
        dev.set_mesh(mesh, rank)
        owned = dev.owned_ids()
        n_owned, n_proxy, _ = dev.local_counts()
        nbr = mesh.neighbor_ids
        proxies = sorted({int(nbr[g, f]) for g in owned for f in range(6)
                          if nbr[g, f] >= 0 and mesh.owner[nbr[g, f]] != rank})
        assert len(proxies) == n_proxy
        local = {int(g): i for i, g in enumerate(owned)}
        local.update({g: n_owned + i for i, g in enumerate(proxies)})
        nbr_local = np.full((n_owned + n_proxy, 6), -1, np.int64)
        for i, g in enumerate(owned):
            for f in range(6):
                if nbr[g, f] >= 0:
                    nbr_local[i, f] = local[int(nbr[g, f])]
        p = oracle.params(nf=7, dx=1.0 / 64)
        U_all = oracle.ic_random(p, 0, mesh.n, 2210)
        U = np.zeros((n_owned + n_proxy, 7, 512))
        U[:n_owned] = U_all[owned]
        plans = {peer: dev.halo_plan(peer) for peer in range(world) if peer != rank}
        cells = {f: slab_cells(f) for f in range(6)}

        def exchange(buf):
            reqs, recvd = [], {}
            for peer, (send, recv) in plans.items():
                msg = np.concatenate([buf[local[int(g)]][:, cells[int(f)]].ravel() for g, f in send]) \
                    if len(send) else np.zeros(0)
                reqs.append(dist.isend(torch.from_numpy(msg.copy()), peer))
                recvd[peer] = torch.zeros(len(recv) * 7 * 192, dtype=torch.float64)
                reqs.append(dist.irecv(recvd[peer], peer))
            for r in reqs:
                r.wait()
            for peer, (_, recv) in plans.items():
                data = recvd[peer].numpy().reshape(len(recv), 7, 192)
                for e, (g, f) in enumerate(recv):
                    buf[local[int(g)]][:, cells[int(f)]] = data[e]

        for _ in range(steps):
            amax = torch.tensor([oracle.max_signal_speed(p, U[:n_owned])], dtype=torch.float64)
            dist.all_reduce(amax, op=dist.ReduceOp.MAX)
            dtdx = ((p.cfl * p.dx) / float(amax.item())) / p.dx
            exchange(U)
            U1 = oracle.stage(p, nbr_local, U, U, 1, dtdx, 0, n_owned)
            exchange(U1)
            U2 = oracle.stage(p, nbr_local, U1, U, 2, dtdx, 0, n_owned)
            exchange(U2)
            U3 = oracle.stage(p, nbr_local, U2, U, 3, dtdx, 0, n_owned)
            U[:n_owned] = U3[:n_owned]
        want, _ = oracle.run(p, nbr, U_all, steps)
        q.put((rank, bool(np.array_equal(U[:n_owned], want[owned])), int(n_owned), int(n_proxy)))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e), 0, 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,periodic,world", [((4, 4, 4), "", 2), ((2, 2, 4), "z", 2), ((3, 2, 2), "xy", 2),
                                                 ((2, 2, 8), "z", 4)])
def test_partitioned_step_equals_single_domain_bitwise(hydro, oracle_lib, dims, periodic, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, periodic, 2, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, ok, n_owned, n_proxy in sorted(results):
        assert ok is True, (rank, ok)
        assert n_owned > 0 and n_proxy > 0
