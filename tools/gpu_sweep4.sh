#!/bin/bash
# 4 GPUs: the reference-format scaling sweep (timing hook on/off) at N = 1, 2, 4 and multi-rank AMR timing.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sweep4
timeout 600 python tools/harness_sweep.py > gpurun_out/sweep4/n1.json 2>gpurun_out/sweep4/n1.err; echo "n1 rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29300 + n)) \
    tools/harness_sweep.py > gpurun_out/sweep4/n$n.json 2>gpurun_out/sweep4/n$n.err; echo "n$n rc=$?"
done
python tools/harness_sweep.py --combine gpurun_out/sweep4/n1.json gpurun_out/sweep4/n2.json gpurun_out/sweep4/n4.json --csv gpurun_out/sweep4/sweep.csv
cat gpurun_out/sweep4/sweep.csv
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29400 + n)) \
    tools/multigpu_check.py --amr ref4 --steps 3 --transport p2p 2>&1 | grep MULTIGPU
done
