#!/bin/bash
# Config 4 (V1309-like binary, 64x64x32 sub-grids, nf 11): strong scaling on 1, 2 and all visible GPUs.
N=$(nvidia-smi -L | wc -l)
for n in 1 2 $N; do
  if [ "$n" = "1" ]; then
    timeout 900 python bench.py --workload binary --no-cpu-baseline --no-e2e > gpurun_out/binary_n1.log 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29700 + n)) bench.py --gpus $n --workload binary --no-cpu-baseline --no-e2e > gpurun_out/binary_n$n.log 2>&1
  fi
  tail -1 gpurun_out/binary_n$n.log > gpurun_out/binary_n$n.json
  echo "binary n=$n $(tail -1 gpurun_out/binary_n$n.log | cut -c1-220)"
done
