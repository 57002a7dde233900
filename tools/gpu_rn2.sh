#!/bin/bash
# rcp_rn all-ones-mantissa fix: selftest bands, 3-D and AMR parity, same-box
# bench against the IEEE-reciprocal build, then the full GPU suite.
out=gpurun_out/rn2.log; rm -f $out
python -c "
from paper_2210_06437_b200 import hydro
d = hydro.CudaDevice(hydro.HydroConfig())
for e in (1000, 4, -4, -60):
    print('selftest emax', e, d.selftest_math(1 << 28, seed=11, emax=e))
" >> $out 2>&1
timeout 300 python tools/parity_3d.py >> $out 2>&1
timeout 300 python tools/amr_diag2.py >> $out 2>&1
for rep in 1 2; do
for lib in paper_2210_06437_b200/libts_hydro.so paper_2210_06437_b200/libts_hydro_ieee.so; do
  for w in "" "--recon minmod" "--workload polytrope"; do
    echo "== bench $(basename $lib) $w" >> $out
    TS_HYDRO_LIB=$PWD/$lib timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-e2e $w >> $out 2>&1
  done
done
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rn2_pytest.log 2>&1
tail -2 gpurun_out/rn2_pytest.log >> $out
