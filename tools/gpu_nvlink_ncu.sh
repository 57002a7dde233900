#!/bin/bash
# 2 GPUs: rank 0 under ncu (NVLink TX/RX user bytes of the fused-push stage
# kernels, single-pass metrics), rank 1 plain; no torchrun so only rank 0 is
# profiled.  Every cross-GPU wait has a deadline, so a replay cannot hang.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export MASTER_ADDR=127.0.0.1 MASTER_PORT=$((29000 + RANDOM % 500)) WORLD_SIZE=2 TS_HYDRO_WAIT_TIMEOUT_MS=20000
M="nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum"
RANK=0 LOCAL_RANK=0 timeout 600 ncu --metrics $M --clock-control none -k regex:stage_kernel --launch-skip 9 --launch-count 6 --csv \
   python tools/nvlink_bytes.py --steps 4 > gpurun_out/nvlink_ncu_r0.log 2>&1 &
P0=$!
RANK=1 LOCAL_RANK=1 timeout 600 python tools/nvlink_bytes.py --steps 4 > gpurun_out/nvlink_ncu_r1.log 2>&1
echo "rank1 rc=$?"
wait $P0; echo "rank0 rc=$?"
grep -E "nvl|stage_kernel|^\{" gpurun_out/nvlink_ncu_r0.log | tail -40
