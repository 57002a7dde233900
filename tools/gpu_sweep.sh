#!/bin/bash
# Config 5: batch sweep at 1, 2 and N GPUs (per-GPU sizes; fused P2P halos at N > 1).
N=$(nvidia-smi -L | wc -l)
SZ="256 1024 4096 16384 65536 262144"
timeout 1200 python tools/sweep.py --sizes $SZ > gpurun_out/sweep_n1.jsonl 2> gpurun_out/sweep_n1.err
for n in 2 $N; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + n)) tools/sweep.py --sizes $SZ > gpurun_out/sweep_n$n.jsonl 2> gpurun_out/sweep_n$n.err
done
wc -l gpurun_out/sweep_n*.jsonl
