#!/bin/bash
# Gravity FMM evidence: parity tests, throughput, coupled hydro + gravity, ncu.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/fmm
timeout 900 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_gravity.py -q > gpurun_out/fmm/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fmm/tests.log
timeout 600 python tools/fmm_bench.py > gpurun_out/fmm/bench.jsonl 2> gpurun_out/fmm/bench.err; echo "bench rc=$?"; cat gpurun_out/fmm/bench.jsonl
timeout 600 python tools/fmm_bench.py --coupled > gpurun_out/fmm/coupled.jsonl 2> gpurun_out/fmm/coupled.err; echo "coupled rc=$?"; cat gpurun_out/fmm/coupled.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fmm/launches.csv \
    python tools/fmm_bench.py --ncu > gpurun_out/fmm/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fmm_ -c 14 -o gpurun_out/fmm/fmm_full \
    python tools/fmm_bench.py --ncu > gpurun_out/fmm/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/fmm/ncu.log
