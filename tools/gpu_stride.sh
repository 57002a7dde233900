#!/bin/bash
# Fused-push A/B: every built library x boundary stride (TS_HYDRO_BSTRIDE) at N GPUs (bench sedov), REPS interleaved.
N=$(nvidia-smi -L | wc -l)
timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('n1 bench', round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],4), 'ms/step')"
p=29830
for rep in $(seq ${REPS:-3}); do
for lib in paper_2210_06437_b200/libts_hydro*.so; do
for st in ${STRIDES:-1 4}; do
  p=$((p + 1))
  r=$(TS_HYDRO_LIB=$lib TS_HYDRO_BSTRIDE=$st timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $p bench.py --gpus $N --no-cpu-baseline --no-e2e $BENCH_ARGS 2>&1 | tail -1 | \
    python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],4), 'ms/step')")
  echo "$(basename $lib) stride $st: $r"
done
done
done
