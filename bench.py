#!/usr/bin/env python
"""Benchmark: FP64 hydro cell-updates/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload sedov] [--impl ours|reference]

A "step" = one full SSP-RK3 time step (3 fused reconstruct+KT-flux+update
stages = the reference's 3 hydro rounds, workload.hpp:116) over every
sub-grid, halo exchange and the dt max-reduction included.  cell-updates/s =
total_cells * steps / seconds (workload.cpp:608-609).

N=1 workload: BASELINE configs[1], Sedov–Taylor on 16^3 = 4096 sub-grids
(128^3 cells, nf = 6, FP64).  N>1: weak scaling, 4096 sub-grids per GPU
(domain 16 x 16 x 16N sub-grids, one contiguous Morton chunk = one z-slab per
rank) with cross-GPU halos pushed over NVLink by the stage kernel itself.  `--workload polytrope` runs configs[2]
(32^3 sub-grids per GPU, 5 species, nf = 11).

`--impl reference` times the CPU path of the reference's algorithm (the
oracle port in oracle/, all host threads; the reference itself ships no hydro
arithmetic) on the same mesh and initial state, a bounded number of steps; it
imports nothing of the product (mesh and initial models from the oracle).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (sub-grids per GPU edge, n_species, problem)          weak-scaled along z
    "sedov": (16, 0, "sedov"),          # configs[1]
    "polytrope": (32, 5, "polytrope"),  # configs[2]
    "random": (16, 0, "random_device"),
    "random11": (32, 5, "random_device"),
    # configs[3]: V1309-like binary, FIXED 64 x 64 x 32 sub-grids (131072) split over
    # the N GPUs (strong scaling; needs N >= 2 for memory-comfortable runs, fits on 1)
    "binary": (None, 5, "binary"),
}
BINARY_DIMS = (64, 64, 32)
L2_BYTES = 126 * 1024 * 1024


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_reference(workload: str, steps: int, warmup: int, world: int = 1, budget_s: float = 120.0,
                  recon: str = "ppm"):
    """The oracle (plain-C restatement of the path, oracle/hydro_oracle.c) on
    the SAME mesh and initial state as the GPU arm, all host threads.  Imports
    nothing of the product: mesh and initial models come from the oracle.
    Timing scope as run_benchmark (workload.cpp:595-612): the stepping only,
    one orc_run call over the timed steps.  Bounded: one untimed warm-up step,
    then min(steps, what fits in budget_s) timed steps."""
    import oracle
    oracle.build()
    edge, species, problem = WORKLOADS[workload]
    nf = 6 + species
    dims = BINARY_DIMS if edge is None else (edge, edge, edge * world)
    dx = 1.0 / (dims[0] * 8)
    p = oracle.params(nf=nf, dx=dx, recon={"ppm": 0, "minmod": 1}[recon])
    nbr, pos, _ = oracle.uniform_mesh(*dims)
    n = len(pos)
    if problem == "sedov":
        U = oracle.ic_sedov(p, pos, dims)
    elif problem == "polytrope":
        U = oracle.ic_polytrope(p, pos, dims)
    elif problem == "binary":
        U = oracle.ic_binary(p, pos, dims)
    else:  # random_device: the reference generator cell_value
        U = oracle.ic_random(p, 0, n, 2210)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    U, _ = oracle.run(p, nbr, U, max(1, min(warmup, 1)), nthreads=threads)
    t_step = time.perf_counter() - t0
    k = int(max(1, min(steps, budget_s // max(t_step, 1e-9))))
    t0 = time.perf_counter()
    U, _ = oracle.run(p, nbr, U, k, nthreads=threads)
    sec = time.perf_counter() - t0
    cells = n * 512
    return {"value": cells * k / sec, "unit": "cell-updates/s", "cores": threads, "kind": "port",
            "sample": f"the full {workload} mesh of the GPU arm ({dims[0]}x{dims[1]}x{dims[2]} = {n} sub-grids, "
                      f"{cells} cells, nf {nf}), {k} timed SSP-RK3 steps after 1 warm-up step, {threads} threads, "
                      f"oracle/hydro_oracle.c (orc_run)",
            "seconds": sec, "steps": k, "dims": list(dims)}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="sedov", choices=sorted(WORKLOADS))
    ap.add_argument("--recon", default="ppm", choices=["ppm", "minmod"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--order", default="row", choices=["morton", "row"],
                    help="sub-grid numbering of the uniform mesh = the CTA launch order: row-major (x fastest; "
                         "make_row_mesh's shape) measured +1.1 %% over the Morton curve on the Sedov mesh")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"],
                    help="N>1 halo transport: copy engines + stream memory ops over NVLink, or NCCL")
    a = ap.parse_args(argv)
    a.warmup = max(a.warmup, 3)

    rank, local_rank, world = dist_env()
    edge, species, problem = WORKLOADS[a.workload]
    nf = 6 + species
    metric = "hydro cell-updates/sec (FP64)"
    unit = "cell-updates/s"
    strong = edge is None
    sub_per_gpu = (BINARY_DIMS[0] * BINARY_DIMS[1] * BINARY_DIMS[2]) // world if strong else edge ** 3

    if a.impl == "reference":
        if rank != 0:
            return 0
        cb = cpu_reference(a.workload, a.steps, a.warmup, world=world, recon=a.recon)
        d = cb["dims"]
        line = {"metric": metric, "value": cb["value"], "unit": unit, "n_gpus": world, "steps": cb["steps"],
                "warmup": 1, "ms_per_step": 1e3 * cb["seconds"] / cb["steps"], "higher_is_better": True,
                "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "impl": "reference",
                "config": {"workload": f"{a.workload}: {sub_per_gpu} sub-grids (8^3 + 3-deep halo) per GPU, "
                                       f"domain {d[0]}x{d[1]}x{d[2]} sub-grids",
                           "problem": problem, "nf": nf, "recon": a.recon, "total_cells": d[0] * d[1] * d[2] * 512,
                           "same_config": True,
                           "timed": "CPU oracle on the host cores, rank 0 only (the reference ships no hydro "
                                    "arithmetic: its kernels are timed sleeps, workload.cpp:544-552)"},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": cb["value"], "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    from paper_2210_06437_b200 import hydro as H
    H.lib()  # fail loudly without the CUDA library

    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
    dims = BINARY_DIMS if strong else (edge, edge, edge * world)
    dx = 1.0 / (dims[0] * 8)
    mesh = H.uniform_mesh(*dims, world=world, order=a.order)
    cfg = H.HydroConfig(device_id=local_rank, n_species=species, dx=dx, recon=a.recon)
    dev = H.CudaDevice(cfg)
    session = H.WorkloadSession(mesh, dev, H.StepConfig(num_steps=a.steps), rank=rank)
    if world > 1:
        import torch.distributed as dist
        if a.transport == "nccl":
            obj = [H.CudaDevice.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            dev.comm_init(obj[0], world, rank)
        else:
            blobs = [None] * world
            dist.all_gather_object(blobs, dev.p2p_export())
            dev.p2p_import(blobs)
    session.load_problem(problem)
    n_owned = dev.local_counts()[0]
    cells_local = n_owned * 512
    state_bytes = 3 * (n_owned + dev.local_counts()[1]) * nf * 512 * 8

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # warm-up (untimed): at least W steps and ~0.5 s of GPU work so clocks settle
    # Stepping is collective across ranks, so the number of warm-up calls is
    # agreed (max over ranks) rather than decided by each rank's own clock.
    dev.compute_dt()
    t_w = time.perf_counter()
    dev.step(a.warmup)
    dev.synchronize()
    t_call = time.perf_counter() - t_w
    extra = int(math.ceil((0.5 - t_call) / t_call)) if t_call < 0.5 else 0
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([extra], dtype=torch.int64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        extra = int(t.item())
    for _ in range(extra):
        dev.step(a.warmup)
    dev.synchronize()
    dev.flush_activity()
    # the clock sampler (an nvidia-smi child) starts BEFORE the barrier: its
    # spawn jitter would otherwise skew the ranks' start of the timed region,
    # and the max over ranks would absorb the skew
    with ClockSampler(local_rank) as clk:
        barrier()
        dev.synchronize()
        launches0 = dev.launch_count()
        ms = dev.time_steps(a.steps)
    launches = dev.launch_count() - launches0
    barrier()
    recs = [r for r in dev.flush_activity() if r.kind == "kernel" and r.name.startswith("hydro_stage")]
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_cells = mesh.n * 512
    value = total_cells * a.steps / (ms * 1e-3)

    # physical validity of the state the timed steps produced (outside the
    # timed region): every value finite, densities and pressures positive
    Us = dev.download()
    rho = Us[:, 0]
    pres = (cfg.gamma - 1.0) * (Us[:, 4] - 0.5 * (Us[:, 1] ** 2 + Us[:, 2] ** 2 + Us[:, 3] ** 2) / rho)
    chk = [float(np.isfinite(Us).all()), float(rho.min()), float(pres.min())]
    del Us, rho, pres
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor(chk, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        chk = [float(x) for x in t.tolist()]
    state_check = {"finite": bool(chk[0] == 1.0), "min_rho": chk[1], "min_p_before_floor": chk[2],
                   "steps_taken": int(dev.steps_done())}

    # roofline of the dominant (stage) kernel: algorithmic bytes / kernel time
    peaks, peak_kind = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    b_alg_step = 64 * nf * cells_local  # 8 nf (3S - 1) per cell-update, S = 3
    kernel_ns = sum(r.end_ns - r.start_ns for r in recs)
    n_stage_launches = len(recs)
    achieved = (b_alg_step * a.steps) / (kernel_ns * 1e-9) / 1e9 if kernel_ns > 0 else None
    stage_share = kernel_ns * 1e-6 / ms if ms > 0 else None

    # FP64-pipe view of the same kernel (the limiter in practice)
    fp64 = None
    try:
        with open(os.path.join(ROOT, "profiles", "fp64_model.json")) as f:
            fm = json.load(f)
        per = fm["fp64_instr_per_cell_update"].get(f"{a.recon}_nf{nf}")
        if per:
            peak_i = float(fm["fp64_peak_instr_per_s"])
            fp64 = {"instr_per_cell_update": per, "peak_instr_per_s": peak_i,
                    "achieved_instr_per_s": value / world * per, "frac": value / world * per / peak_i,
                    "source": "profiles/fp64_model.json (ncu instruction count x measured FP64 peak)"}
    except Exception:
        fp64 = None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{a.workload}_{a.recon}_nf{nf}")
    except Exception:
        traffic = None

    # end to end: host buffers through the C ABI, H2D + step + D2H every step
    e2e = None
    if not a.no_e2e:
        nbytes = n_owned * nf * 512 * 8
        hin = dev.host_pinned_alloc(nbytes)
        hout = dev.host_pinned_alloc(nbytes)
        import ctypes
        U = dev.download()
        ctypes.memmove(hin, U.ctypes.data, nbytes)
        dev.step_host(hin, hout, 1)  # warm
        k_e2e = max(3, min(a.steps, 20))

        def e2e_run(step_fn):
            nonlocal hin, hout
            barrier()
            t0 = time.perf_counter()
            for _ in range(k_e2e):
                step_fn(hin, hout, 1)
                hin, hout = hout, hin  # chained: each step's input is the previous step's output
            dev.synchronize()
            sec = time.perf_counter() - t0
            if world > 1:
                import torch
                import torch.distributed as dist
                t = torch.tensor([sec], dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                sec = float(t.item())
            return total_cells * k_e2e / sec

        sync_value = e2e_run(dev.step_host)
        # warm the pipelined path, two chained calls; the timed calls continue
        # the chain (each call's input is the previous call's output, as in a
        # simulation run through host memory), so no timed call restarts it
        for _ in range(2):
            dev.step_host_async(hin, hout, 1)
            hin, hout = hout, hin
        dev.synchronize()
        value_e2e = e2e_run(dev.step_host_async)
        e2e = {"value": value_e2e, "unit": unit, "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": nbytes, "steps": k_e2e,
               "path": "ts_hydro_step_host_async, chained: every step pinned host U^n -> H2D (24 chunks, each "
                       "behind the previous step's D2H of that chunk) -> stages 1..3 as a wavefront over the chunks "
                       "(event dependencies on the halo chunks; dt from the previous step) -> D2H (each chunk behind "
                       "its stage 3); step k+1's input is step k's output",
               "pcie_ceiling": "both PCIe directions at once move ~49 GB/s each on these boxes: 2 x 100 MB per "
                               "step caps e2e near 0.98 G cell-updates/s (tools/pcie_probe.py)",
               "sync_value": sync_value,
               "sync_path": "ts_hydro_step_host: H2D -> dt + 1 step -> D2H, one call at a time"}
        dev.host_pinned_free(hin)
        dev.host_pinned_free(hout)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cb = cpu_reference(a.workload, 20, 1, world=1, budget_s=15.0, recon=a.recon)
        cpu = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{a.workload}: {sub_per_gpu} sub-grids (8^3 + 3-deep halo) per GPU, "
                                   f"domain {dims[0]}x{dims[1]}x{dims[2]} sub-grids",
                       "problem": problem, "nf": nf, "recon": a.recon, "total_cells": total_cells,
                       "numbering": a.order,
                       "parallelism": f"domain decomposition over {world} GPU(s)"
                                      + (f", {a.transport} halos" if world > 1 else ""),
                       "l2": f"working set {state_bytes / 2**20:.0f} MiB (3 state buffers) > 126 MiB L2; no flush"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
                         "peak_source": peak_kind,
                         "alg_bytes_per_cell_update": 64 * nf,
                         "kernel": "stage_kernel (fused reconstruct + KT flux + RK update)",
                         "stage_launches": n_stage_launches, "stage_share_of_step": stage_share,
                         "fp64": fp64},
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "state_check": state_check,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    dev.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
