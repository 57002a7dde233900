#!/bin/bash
# nf 11: species-accumulator ring A/B (parity, throughput, DRAM bytes per launch).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_amr.py -x -q -k "species or config3 or config4 or config5 or every_field or dataflow or amr_steps" > gpurun_out/t_nf11.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_nf11.log
rm -f gpurun_out/nf11.log
for rep in 1 2; do
for ring in 1 0; do
  echo "== ring $ring" >> gpurun_out/nf11.log
  TS_HYDRO_SCR_RING=$ring timeout 300 python bench.py --workload polytrope --steps 10 --warmup 3 --no-cpu-baseline --no-e2e >> gpurun_out/nf11.log 2>&1
done
done
python tools/variants.py gpurun_out/nf11.log
for ring in 1 0; do
TS_HYDRO_SCR_RING=$ring timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:stage_kernel --launch-skip 12 --launch-count 3 --csv python bench.py --workload polytrope --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_nf11_ring$ring.csv 2>&1; echo "ncu ring$ring rc=$?"
done
