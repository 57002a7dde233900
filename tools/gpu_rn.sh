#!/bin/bash
# rcp / sqrt rounding investigation: selftest (near-one mantissas), 3-D parity
# and same-box Sedov bench for every library variant.
out=gpurun_out/rn.log; rm -f $out
for lib in paper_2210_06437_b200/libts_hydro.so paper_2210_06437_b200/libts_hydro_*.so; do
  echo "== $(basename $lib)" >> $out
  TS_HYDRO_LIB=$PWD/$lib timeout 120 python -c "
from paper_2210_06437_b200 import hydro
d = hydro.CudaDevice(hydro.HydroConfig())
for e in (4, -4, -60):
    print('selftest emax', e, d.selftest_math(1 << 26, seed=11, emax=e))
" >> $out 2>&1
  TS_HYDRO_LIB=$PWD/$lib timeout 300 python tools/parity_3d.py >> $out 2>&1
done
for rep in 1 2; do
for lib in paper_2210_06437_b200/libts_hydro.so paper_2210_06437_b200/libts_hydro_ieee.so paper_2210_06437_b200/libts_hydro_rnfix.so paper_2210_06437_b200/libts_hydro_ircp.so paper_2210_06437_b200/libts_hydro_isqrt.so; do
  echo "== bench $(basename $lib)" >> $out
  TS_HYDRO_LIB=$PWD/$lib timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-e2e >> $out 2>&1
done
done
