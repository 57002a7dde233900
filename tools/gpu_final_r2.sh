#!/bin/bash
# End-of-round evidence at HEAD (one GPU): the standard evidence run, the
# self-check build over the suite, and ncu captures of the minmod / nf 11
# stage kernels for their FP64 instruction counts.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
tag=${1:-r2e}
bash tools/gpu_evidence.sh $tag
bash tools/gpu_check.sh > gpurun_out/${tag}_selfcheck.txt 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 3 -c 3 -o gpurun_out/${tag}_stage_minmod $B --recon minmod > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 3 -c 3 -o gpurun_out/${tag}_stage_poly $B --workload polytrope > /dev/null 2>&1
echo final done
