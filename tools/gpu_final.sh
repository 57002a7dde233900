#!/bin/bash
# Round evidence after the AMR + IEEE-reciprocal change: the standard evidence
# run plus the AMR throughput lines.
tag=${1:-r1h}
bash tools/gpu_evidence.sh $tag
timeout 300 python tools/amr_bench.py > gpurun_out/${tag}_amr_bench.json 2>&1
timeout 300 python tools/amr_bench.py --species 5 --base 24 --refined 8 > gpurun_out/${tag}_amr_bench_nf11.json 2>&1
python tools/ncu_summary.py gpurun_out/${tag}_stage.ncu-rep > gpurun_out/${tag}_stage_summary.txt 2>&1 || true
echo final done
