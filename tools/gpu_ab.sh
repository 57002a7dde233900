#!/bin/bash
# Same-box A/B of every built library variant, interleaved twice (bench only).
rm -f gpurun_out/variants.log
for rep in 1 2; do
for lib in paper_2210_06437_b200/libts_hydro*.so; do
  for w in "--workload sedov" "--workload sedov --recon minmod" $EXTRA_WORKLOADS; do
    echo "== $(basename $lib) $w" >> gpurun_out/variants.log
    TS_HYDRO_LIB=$lib timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-e2e $w >> gpurun_out/variants.log 2>&1
  done
done
done
