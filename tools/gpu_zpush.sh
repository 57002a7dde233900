#!/bin/bash
# In-z-sweep slab push (TS_ZPUSH) vs the post-sweep push: world-4 parity and weak scaling A/B.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
port() { echo $((29100 + RANDOM % 800)); }
ZP=paper_2210_06437_b200/libts_hydro_zp.so
for dims in "4 4 8" "4 4 4 --periodic xyz --species 5"; do
  TS_HYDRO_LIB=$ZP timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $(port) \
    tools/multigpu_check.py --dims $dims --transport p2p --steps 4 2>&1 | grep -h "MULTIGPU" | sed 's/^/[zp] /'
done
for rep in 1 2; do
  for lib in paper_2210_06437_b200/libts_hydro.so $ZP; do
    for n in 1 2 4; do
      if [ $n = 1 ]; then
        r=$(TS_HYDRO_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3))")
      else
        r=$(TS_HYDRO_LIB=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $(port) \
            bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3))")
      fi
      echo "$(basename $lib) n$n $r"
    done
  done
done
