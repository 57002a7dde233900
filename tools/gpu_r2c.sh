#!/bin/bash
# e2e gate check, TMA variant parity + A/B, ncu source capture of the stage kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "pipelined" > gpurun_out/t_pipe.log 2>&1; echo "pipe rc=$?"
TS_HYDRO_LIB=$PWD/paper_2210_06437_b200/libts_hydro_tma.so timeout 900 python -m pytest tests/test_gpu.py -x -q -k "random_state or sedov_4096 or config1 or each_rk or dataflow or dropin or smooth_bump" > gpurun_out/t_tma.log 2>&1; echo "tma tests rc=$?"
rm -f gpurun_out/variants.log
for rep in 1 2; do
for lib in paper_2210_06437_b200/libts_hydro.so paper_2210_06437_b200/libts_hydro_tma.so; do
  echo "== $(basename $lib)" >> gpurun_out/variants.log
  TS_HYDRO_LIB=$PWD/$lib timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e >> gpurun_out/variants.log 2>&1
done
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage_kernel --launch-skip 30 --launch-count 3 -o gpurun_out/stage_src -f python bench.py --steps 5 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_src.log 2>&1; echo "ncu rc=$?"
TS_HYDRO_LIB=$PWD/paper_2210_06437_b200/libts_hydro_tma.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage_kernel --launch-skip 30 --launch-count 3 -o gpurun_out/stage_src_tma -f python bench.py --steps 5 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_src_tma.log 2>&1; echo "ncu tma rc=$?"
python tools/variants.py gpurun_out/variants.log
