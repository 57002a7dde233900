#!/bin/bash
# Evidence run for profiles/: full GPU tests, default bench, ncu launch list
# and a full ncu capture of the fused stage kernel (one GPU).
# usage: bash tools/gpu_evidence.sh <tag>
tag=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${tag}_smi.txt
nproc > gpurun_out/${tag}_nproc.txt; lscpu | grep "Model name" >> gpurun_out/${tag}_nproc.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${tag}_pytest_gpu.log 2>&1
tail -2 gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 600 python bench.py --recon minmod --no-cpu-baseline > gpurun_out/${tag}_bench_minmod.json 2>&1
timeout 600 python bench.py --workload polytrope --no-cpu-baseline > gpurun_out/${tag}_bench_poly.json 2>&1
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv $B > /dev/null 2>&1
$B > gpurun_out/${tag}_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 3 -c 3 -o gpurun_out/${tag}_stage $B > gpurun_out/${tag}_ncu.log 2>&1
echo "evidence done"
