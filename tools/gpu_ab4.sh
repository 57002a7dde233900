#!/bin/bash
# A/B of the N-GPU transports / dt-wait modes (bench sedov), plus the multi-GPU parity tests.
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1
tail -1 gpurun_out/ab_pytest.log
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 bench.py --gpus $N --no-cpu-baseline --no-e2e ${@:2} 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['parallelism'], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],4), 'ms/step')"; }
echo "p2p device-wait: $(run 29701 --transport p2p)"
echo "p2p stream-wait: $(TS_HYDRO_DT_WAIT=stream run 29702 --transport p2p)"
echo "nccl:            $(run 29703 --transport nccl)"
echo "p2p polytrope:   $(run 29704 --transport p2p --workload polytrope)"
