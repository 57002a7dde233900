#!/bin/bash
# Multi-GPU round (gpurun --gpus N): NCCL parity tests, then the weak-scaling bench at N.
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1
tail -3 gpurun_out/pytest_multi.log
for n in 1 $N; do
  if [ "$n" = "1" ]; then
    timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 29533 bench.py --gpus $n --no-cpu-baseline > gpurun_out/bench_n$n.log 2>&1
  fi
  tail -1 gpurun_out/bench_n$n.log | cut -c1-400
done
echo done
