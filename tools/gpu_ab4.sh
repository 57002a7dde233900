#!/bin/bash
# A/B of the N-GPU transports / dt-wait modes (bench sedov), plus the multi-GPU parity tests.
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > gpurun_out/ab_pytest.log 2>&1
tail -1 gpurun_out/ab_pytest.log
for t in p2p nccl; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2969$N \
    tools/multigpu_check.py --dims 4 4 16 --periodic z --transport $t 2>&1 | grep -E "MULTIGPU|Error|mismatch" | head -3
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2968$N \
    tools/multigpu_check.py --dims 3 5 3 --periodic xy --species 1 --transport $t 2>&1 | grep -E "MULTIGPU|Error|mismatch" | head -3
done
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 bench.py --gpus $N --no-cpu-baseline --no-e2e ${@:2} 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['parallelism'], round(d['value']/1e9,3), 'G/s', round(d['ms_per_step'],4), 'ms/step')"; }
echo "p2p fused push:  $(run 29701 --transport p2p)"
echo "p2p copy-engine halos: $(TS_HYDRO_HALO=ce run 29705 --transport p2p)"
echo "nccl:            $(run 29703 --transport nccl)"
echo "p2p polytrope:   $(run 29704 --transport p2p --workload polytrope)"
