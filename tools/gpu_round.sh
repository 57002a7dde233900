#!/bin/bash
# one GPU round: parity tests, then bench variants (usage: bash tools/gpu_round.sh)
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for v in "" _minb4 _minb8; do
  for w in "--workload sedov" "--workload sedov --recon minmod" "--workload polytrope"; do
    echo "== lib$v $w" >> gpurun_out/variants.log
    TS_HYDRO_LIB=paper_2210_06437_b200/libts_hydro$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $w >> gpurun_out/variants.log 2>&1
  done
done
echo done
