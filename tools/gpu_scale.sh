#!/bin/bash
# Weak-scaling runs on all visible GPUs: sedov (config 2 per GPU) and polytrope (config 3).
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/scale_pytest.log 2>&1
tail -1 gpurun_out/scale_pytest.log
for w in sedov polytrope; do
  for n in 1 2 $N; do
    if [ "$n" = "1" ]; then
      timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/scale_${w}_n1.log 2>&1
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29600 + n)) bench.py --gpus $n --workload $w --no-cpu-baseline --no-e2e > gpurun_out/scale_${w}_n$n.log 2>&1
    fi
    echo "$w n=$n $(tail -1 gpurun_out/scale_${w}_n$n.log | cut -c1-160)"
  done
done
