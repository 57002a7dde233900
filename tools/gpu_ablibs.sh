#!/bin/bash
# Same-box A/B of named library variants (bench sedov PPM, interleaved REPS times).
# usage: LIBS="base minb8 fp8" [REPS=2] [WL="--workload sedov"] bash tools/gpu_ablibs.sh [bench args]
mkdir -p gpurun_out
out=gpurun_out/ablibs.log
rm -f $out
for rep in $(seq ${REPS:-2}); do
  for v in $LIBS; do
    lib=paper_2210_06437_b200/libts_hydro_$v.so
    [ "$v" = base ] && lib=paper_2210_06437_b200/libts_hydro.so
    echo "== $v rep $rep" >> $out
    TS_HYDRO_LIB=$lib timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-e2e ${WL:---workload sedov} "$@" >> $out 2>&1
  done
done
python tools/variants.py $out
