#!/bin/bash
# Gravity FMM evidence: parity tests, throughput, ncu of the leaf kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/fmm
timeout 900 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_gravity.py -q > gpurun_out/fmm/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fmm/tests.log
timeout 600 python tools/fmm_bench.py > gpurun_out/fmm/bench.jsonl 2> gpurun_out/fmm/bench.err; echo "bench rc=$?"; cat gpurun_out/fmm/bench.jsonl
#TS_HYDRO_FMM_NOSPLIT=1 timeout 600 python tools/fmm_bench.py > gpurun_out/fmm/bench_nosplit.jsonl 2>&1; echo "nosplit rc=$?"; cat gpurun_out/fmm/bench_nosplit.jsonl
#timeout 600 ncu --set full --clock-control none --import-source on -k regex:fmm_ -c 12 -o gpurun_out/fmm/fmm_full \
#    python tools/fmm_bench.py --ncu > gpurun_out/fmm/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/fmm/ncu.log
