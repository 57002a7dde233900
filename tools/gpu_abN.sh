#!/bin/bash
# Same-box A/B of every built library variant at N GPUs (bench sedov, interleaved twice).
N=$(nvidia-smi -L | wc -l)
for rep in 1 2; do
for lib in paper_2210_06437_b200/libts_hydro*.so; do
  r=$(TS_HYDRO_LIB=$lib timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29900 + rep)) bench.py --gpus $N --no-cpu-baseline --no-e2e $@ 2>&1 | tail -1 | \
      python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],4), 'ms/step')")
  echo "$(basename $lib) $r"
done
done
