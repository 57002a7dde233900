cd "${GRAFT_REPO_ROOT:-/root/repo}"
port() { echo $((29100 + RANDOM % 800)); }
export TS_HYDRO_DT=tail
for k in 20 100 20 100; do
  r=$(timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $(port) \
        bench.py --gpus 2 --steps $k --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
        python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['ms_per_step'],4))")
  echo "steps $k n2 $r"
  r=$(timeout 300 python bench.py --steps $k --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
        python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), round(d['ms_per_step'],4))")
  echo "steps $k n1 $r"
done
