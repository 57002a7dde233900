#!/bin/bash
# Hydro + self-gravity weak scaling on 1 / 2 / 4 GPUs of one box (tools/gravity_scale.py).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/gscale
timeout 600 python tools/gravity_scale.py > gpurun_out/gscale/n1.json 2> gpurun_out/gscale/n1.err; echo "n1 rc=$?"; cat gpurun_out/gscale/n1.json
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n)) \
     tools/gravity_scale.py > gpurun_out/gscale/n$n.json 2> gpurun_out/gscale/n$n.err; echo "n$n rc=$?"; cat gpurun_out/gscale/n$n.json
done
