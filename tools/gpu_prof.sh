#!/bin/bash
# ncu capture of the stage kernel (one GPU): bash tools/gpu_prof.sh <tag> [bench args]
tag=$1; shift
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $*"
$B > gpurun_out/prof_${tag}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 3 -c 3 -o gpurun_out/prof_${tag} $B > gpurun_out/prof_${tag}_ncu.log 2>&1
echo "rc=$?"
