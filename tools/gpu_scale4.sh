#!/bin/bash
# 4 GPUs of one box: world-4 parity (all transports) and weak scaling N = 1, 2, 4.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/scale4
port() { echo $((29100 + RANDOM % 800)); }
for tr in p2p p2p-ce nccl; do
  for dims in "4 4 8" "4 4 4 --periodic xyz --species 5"; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $(port) \
      tools/multigpu_check.py --dims $dims --transport $tr > gpurun_out/scale4/check_${tr}_$(echo $dims | tr ' ' '_').log 2>&1
    echo "world4 $tr [$dims] rc=$? $(grep -h 'MULTIGPU' gpurun_out/scale4/check_${tr}_$(echo $dims | tr ' ' '_').log)"
  done
done
for w in sedov polytrope; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/scale4/${w}_n1.json 2>/dev/null; echo "$w n1 rc=$?"
  for n in 2 4; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $(port) \
      bench.py --gpus $n --workload $w --steps 20 --warmup 5 --no-e2e > gpurun_out/scale4/${w}_n$n.json 2>/dev/null; echo "$w n$n rc=$?"
  done
done
python - <<'PY'
import json
for w in ("sedov", "polytrope"):
    v = {}
    for n in (1, 2, 4):
        try:
            d = json.loads([l for l in open(f"gpurun_out/scale4/{w}_n{n}.json") if l.startswith("{")][-1])
            v[n] = d["value"]
        except Exception as e:
            v[n] = None
    if v[1]:
        print(w, {n: (round(x / 1e9, 3), round(x / (n * v[1]), 4) if x else None) for n, x in v.items() if x})
PY
