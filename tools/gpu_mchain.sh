#!/bin/bash
# 2 GPUs: multi-rank step chaining (TS_HYDRO_DT=tail + TS_HYDRO_MCHAIN) A/B
# against the default one-thread dt kernel; world-2 parity of each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
port() { echo $((29100 + RANDOM % 800)); }
for e in "TS_HYDRO_DT=kernel" "TS_HYDRO_DT=tail TS_HYDRO_MCHAIN=1"; do
  for dims in "4 4 8" "4 4 4 --periodic xyz --species 5"; do
    env $e timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $(port) \
      tools/multigpu_check.py --dims $dims --transport p2p --steps 6 2>&1 | grep -h MULTIGPU | sed "s/^/[$e] /"
  done
done
for rep in 1 2; do
  for e in "TS_HYDRO_DT=kernel" "TS_HYDRO_DT=tail TS_HYDRO_MCHAIN=0" "TS_HYDRO_DT=tail TS_HYDRO_MCHAIN=1"; do
    r=$(env $e timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $(port) \
        bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
        python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3))")
    echo "$e sedov n2 $r"
  done
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline | tail -1 | \
  python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('n1', round(d['value']/1e9,3))"
