#!/bin/bash
# Same-box N=1 bench + per-rank kernel timelines at 1 and N ranks (activity records).
N=$(nvidia-smi -L | wc -l)
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | cut -c1-200
timeout 300 python tools/timeline.py --steps 2 "$@" > gpurun_out/timeline_n1.txt 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29811 \
  tools/timeline.py --steps 2 "$@" > gpurun_out/timeline_n$N.txt 2>&1
grep -E "^rank" gpurun_out/timeline_n1.txt gpurun_out/timeline_n$N.txt
