#!/bin/bash
# ncu --set full of the stage kernels (HEAD, row numbering) and the gravity P2P kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/ncu2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stage_kernel --launch-skip 30 --launch-count 3 \
  -o gpurun_out/ncu2/stage_full -f python bench.py --steps 5 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu2/stage.log 2>&1; echo "stage rc=$?"
timeout 600 ncu --set full --clock-control none -k regex:p2p_kernel --launch-skip 3 --launch-count 1 \
  -o gpurun_out/ncu2/p2p_full -f python tools/gravity_bench.py > gpurun_out/ncu2/p2p.log 2>&1; echo "p2p rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu2/launches.csv 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fmm_ -c 14 -o gpurun_out/ncu2/fmm_full -f \
    python tools/fmm_bench.py --ncu > gpurun_out/ncu2/fmm.log 2>&1; echo "fmm rc=$?"
