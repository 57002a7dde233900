#!/bin/bash
# Hydro + self-gravity at 4 GPUs: FMM merged part launch on / off, same box, twice.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2; do for m in 0 1; do
  r=$(TS_HYDRO_FMM_MERGE=$m timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) \
     tools/gravity_scale.py 2>/dev/null | grep '^{')
  echo "merge=$m $r"
done; done
