#!/bin/bash
# 2 GPUs: NVLink data counters around the fused halo push vs the halo plan; 2-GPU parity tests; scaling points.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for tr in p2p p2p-ce; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) tools/nvlink_bytes.py --transport $tr > gpurun_out/nvlink_$tr.log 2>&1; echo "nvlink $tr rc=$?"
grep '^{' gpurun_out/nvlink_$tr.log
done
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q > gpurun_out/t_multirank2.log 2>&1; echo "multirank rc=$?"; tail -2 gpurun_out/t_multirank2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench n2 rc=$?"
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err; echo "bench n1 rc=$?"
