#!/bin/bash
# Multi-GPU parity tests, then Sedov/polytrope weak scaling at 1, 2 and all
# visible GPUs for each setting in ENVS (default: dataflow off / on).
N=$(nvidia-smi -L | wc -l)
ENVS=${ENVS:-"TS_HYDRO_FLOW=0 TS_HYDRO_FLOW=1"}
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -x -p no:cacheprovider > gpurun_out/scale_pytest.log 2>&1
tail -1 gpurun_out/scale_pytest.log
for w in ${WORKLOADS:-sedov}; do
for e in $ENVS; do
  for n in 1 2 $N; do
    if [ "$n" = "1" ]; then
      env $e timeout 600 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/scale_${w}_${e}_n1.log 2>&1
    else
      env $e timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29600 + n)) bench.py --gpus $n --workload $w --no-cpu-baseline --no-e2e > gpurun_out/scale_${w}_${e}_n$n.log 2>&1
    fi
    echo "$w $e n=$n $(tail -1 gpurun_out/scale_${w}_${e}_n$n.log | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e9,3), "G/s", round(d["ms_per_step"],4), "ms/step")' 2>&1 | tail -1)"
  done
done
done
