#!/bin/bash
# Round-end scaling evidence on all visible GPUs: Sedov / polytrope weak
# scaling and the binary (config 4) strong scaling at 1, 2 and N GPUs.
N=$(nvidia-smi -L | wc -l)
for w in sedov polytrope binary; do
  for n in 1 2 $N; do
    if [ "$n" = "1" ]; then
      timeout 900 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/sc_${w}_n1.log 2>&1
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29700 + n)) bench.py --gpus $n --workload $w --no-cpu-baseline --no-e2e > gpurun_out/sc_${w}_n$n.log 2>&1
    fi
    tail -1 gpurun_out/sc_${w}_n$n.log > gpurun_out/sc_${w}_n$n.json
    echo "$w n=$n $(python3 -c "import json; d=json.load(open('gpurun_out/sc_${w}_n$n.json')); print(round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],3), 'ms', d['clocks'])" 2>&1 | tail -1)"
  done
done
