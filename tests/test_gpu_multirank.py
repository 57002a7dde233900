"""Cross-rank halo exchange parity: runs tools/multigpu_check.py under
torchrun with world size 2 — one rank per GPU when the box has two (gpurun
--gpus 2), and always both ranks on cuda:0 (two processes sharing one GPU
through CUDA IPC, time-sliced by the driver), so the fused in-kernel slab push
(p2p) and the copy-engine exchange (p2p-ce) run on a one-GPU box too.  NCCL
refuses two ranks on one device, so its cases need two GPUs."""
import os
import socket
import subprocess
import sys

import pytest

from tests.conftest import ROOT

pytestmark = pytest.mark.gpu


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(script_args, timeout, nproc=2, env=None):
    """torchrun world `nproc` on 127.0.0.1; a rendezvous port taken between
    picking and binding it (EADDRINUSE) is retried with a fresh one."""
    env = dict(os.environ, **(env or {}))
    for _ in range(3):
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(nproc),
               "--master-addr", "127.0.0.1", "--master-port", str(_port()),
               os.path.join(ROOT, "tools", "multigpu_check.py"), *script_args]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
        if "EADDRINUSE" not in r.stderr:
            return r
    return r


@pytest.mark.parametrize("transport", ["p2p", "p2p-ce", "nccl"])
@pytest.mark.parametrize("args", [["--dims", "4", "4", "8"], ["--dims", "2", "4", "4", "--periodic", "xyz", "--species", "5"],
                                  ["--dims", "4", "2", "6", "--recon", "minmod", "--steps", "2"],
                                  # ragged Morton chunks: x- and y-face slabs, several foreign faces per sub-grid
                                  ["--dims", "3", "3", "3"],
                                  ["--dims", "5", "3", "2", "--periodic", "x", "--recon", "minmod", "--species", "2"]])
def test_two_gpu_step_is_bitwise_equal_to_single_gpu(args, transport):
    n = _gpus()
    if n < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    r = _torchrun([*args, "--transport", transport], 600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTIGPU OK" in r.stdout


SAME_DEVICE_MESHES = [["--dims", "4", "4", "8"],
                      ["--dims", "2", "4", "4", "--periodic", "xyz", "--species", "5"],
                      ["--dims", "5", "3", "2", "--periodic", "x", "--recon", "minmod", "--species", "2"]]


@pytest.mark.parametrize("transport", ["p2p", "p2p-ce"])
@pytest.mark.parametrize("args", SAME_DEVICE_MESHES)
def test_two_ranks_on_one_gpu_bitwise_equal_to_single_rank(args, transport):
    """World 2 on one GPU: rank-partitioned steps (Morton chunks, proxies,
    slab push / copy-engine exchange, dt all-reduce across the ranks) equal
    the one-rank run bitwise — the partition invariance of
    test_workload.cpp:317-331 / 448-464 on the cross-rank code path."""
    if _gpus() < 1:
        pytest.skip("needs a GPU")
    r = _torchrun([*args, "--transport", transport, "--same-device"], 600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTIGPU OK" in r.stdout


@pytest.mark.parametrize("env", [{"TS_HYDRO_DT": "kernel"}, {"TS_HYDRO_MCHAIN": "0"}])
@pytest.mark.parametrize("args", SAME_DEVICE_MESHES[:2])
def test_two_ranks_on_one_gpu_dt_variants(args, env):
    """The default fused-P2P step gathers dt in stage 3's tail and chains the
    next stage 1 behind it (StageArgs::cnt_gather); the one-thread dt kernel
    and the unchained tail stay bitwise equal to one rank too."""
    if _gpus() < 1:
        pytest.skip("needs a GPU")
    r = _torchrun([*args, "--transport", "p2p", "--same-device", "--steps", "5"], 600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTIGPU OK" in r.stdout


@pytest.mark.parametrize("order", ["stage", "grid"])
@pytest.mark.parametrize("args", [["--dims", "4", "4", "4"], ["--dims", "3", "2", "4", "--periodic", "xyz", "--species", "2"]])
def test_dropin_steps_across_ranks_bitwise_equal_to_single_rank(args, order):
    """The per-sub-grid drop-in (ts_hydro_launch_stage) on two ranks: every
    sub-grid's stage launched alone on a rotating stream, scrambled, no host
    barrier; the boundary sub-grids' halos move by the fused in-kernel push;
    batched steps before and after.  Bitwise equal to one rank, equal dt."""
    extra = ["--same-device"] if _gpus() < 2 else []
    r = _torchrun([*args, "--transport", "p2p", "--dropin", order, "--steps", "4", *extra], 600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTIGPU OK" in r.stdout


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("args", [["--dims", "4", "4", "4"], ["--dims", "3", "5", "2"]])
def test_self_gravity_across_ranks_bitwise_equal_to_single_rank(args, transport):
    """The FMM over the global tree on two GPUs (densities all-gathered over
    NCCL, each rank evaluating its own leaves and their ancestors'
    expansions), and hydro + self-gravity steps: bitwise equal to one rank."""
    if _gpus() < 2:
        pytest.skip("needs 2 GPUs (NCCL refuses two ranks on one device)")
    r = _torchrun([*args, "--transport", transport, "--gravity"], 600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTIGPU OK" in r.stdout


@pytest.mark.parametrize("extra", [["--transport", "p2p"], ["--transport", "p2p-ce"],
                                   ["--transport", "p2p", "--dropin", "grid"]])
def test_eight_ranks_on_one_gpu_bitwise_equal_to_single_rank(extra):
    """World 8 — the driver's largest scaling run — as eight processes sharing
    one GPU through CUDA IPC: every peer mask, flag array and push table at
    eight ranks, batched and drop-in steps, bitwise equal to one rank."""
    r = _torchrun(["--dims", "4", "4", "8", *extra, "--same-device"], 600, nproc=8)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTIGPU OK world=8" in r.stdout


@pytest.mark.parametrize("transport", ["p2p", "p2p-ce"])
def test_mismatch_on_one_gpu_fails_instead_of_hanging(transport):
    if _gpus() < 1:
        pytest.skip("needs a GPU")
    r = _torchrun(["--mismatch", "--transport", transport, "--same-device"], 300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MISMATCH DETECTED" in r.stdout


@pytest.mark.parametrize("transport", ["p2p", "p2p-ce"])
def test_mismatched_collective_call_fails_instead_of_hanging(transport):
    """Stepping is collective: a rank that makes one call too many must get
    TS_ECOMM from the cross-GPU wait deadline, not spin the GPU forever."""
    n = _gpus()
    if n < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    r = _torchrun(["--mismatch", "--transport", transport], 300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MISMATCH DETECTED" in r.stdout


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
@pytest.mark.parametrize("args", [["--amr", "lshape", "--steps", "3"],
                                  ["--amr", "ref4", "--steps", "3", "--species", "5"],
                                  ["--amr", "ref4", "--steps", "2", "--recon", "minmod"]])
def test_multi_rank_amr_bitwise_equal_to_single_rank(args, transport):
    """Coarse-fine AMR partitioned over two ranks (the reference's Morton deal
    of the leaves, workload.cpp:298-323; ghost leaves refreshed whole before
    every stage; dt reduced over the ranks): bitwise the one-rank run.  On one
    GPU the two ranks share it (CUDA IPC, copy-engine transport); NCCL needs
    two GPUs."""
    n = _gpus()
    if n < 1 or (transport == "nccl" and n < 2):
        pytest.skip("needs a GPU (NCCL: two)")
    extra = ["--same-device"] if n < 2 else []
    r = _torchrun([*args, "--transport", transport, *extra], 600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MULTIGPU OK" in r.stdout
