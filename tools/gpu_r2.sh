#!/bin/bash
# Round-2 GPU check: new parity tests, cross-rank on one GPU, adapter, bench.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "${K:-dropin or compute_dt_after or full_size or config5 or each_rk}" > gpurun_out/t_gpu.log 2>&1; echo "t_gpu rc=$?"
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q -k "one_gpu" > gpurun_out/t_multi.log 2>&1; echo "t_multi rc=$?"
timeout 300 python -m pytest tests/test_adapter.py tests/test_gpu_device.py -x -q > gpurun_out/t_adapter.log 2>&1; echo "t_adapter rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -3 gpurun_out/t_gpu.log gpurun_out/t_multi.log gpurun_out/t_adapter.log
