#!/bin/bash
# Same-box A/B of library variants at 2 and N GPUs (Sedov), interleaved twice.
N=$(nvidia-smi -L | wc -l)
for rep in 1 2; do
for lib in paper_2210_06437_b200/libts_hydro*.so; do
  for n in 2 $N; do
    r=$(TS_HYDRO_LIB=$lib timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29820 + n + rep)) bench.py --gpus $n --no-cpu-baseline --no-e2e ${WL:-} 2>&1 | tail -1 | \
        python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s", round(d["ms_per_step"],4), "ms")' 2>&1 | tail -1)
    echo "$(basename $lib) n=$n $r"
  done
done
done
