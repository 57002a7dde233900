#!/bin/bash
# Full GPU suite + bench (N=1) + reference arm.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/t_all.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
TS_HYDRO_H2D_GATE=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_nogate.json 2> gpurun_out/bench_nogate.err; echo "bench nogate rc=$?"
tail -15 gpurun_out/t_all.log
