#!/bin/bash
# One GPU round: parity tests on the default library, then the bench on every
# built library variant (paper_2210_06437_b200/libts_hydro*.so).
# usage: bash tools/gpu_round.sh [workload-args ...]   (default: sedov ppm, sedov minmod, polytrope)
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
rm -f gpurun_out/variants.log
for lib in paper_2210_06437_b200/libts_hydro*.so; do
  for w in "--workload sedov" "--workload sedov --recon minmod" "--workload polytrope"; do
    echo "== $(basename $lib) $w" >> gpurun_out/variants.log
    TS_HYDRO_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $w >> gpurun_out/variants.log 2>&1
  done
done
echo done
