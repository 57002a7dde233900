#!/bin/bash
# Same-box A/B of environment settings (bench only, interleaved twice).
# usage: ENVS="TS_HYDRO_FLOW=0 TS_HYDRO_FLOW=1" bash tools/gpu_abenv.sh [bench args]
rm -f gpurun_out/variants.log
for rep in 1 2; do
for e in $ENVS; do
  for w in "--workload sedov" "--workload sedov --recon minmod" $EXTRA_WORKLOADS; do
    echo "== $e $w" >> gpurun_out/variants.log
    env $e timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-e2e $w "$@" >> gpurun_out/variants.log 2>&1
  done
done
done
