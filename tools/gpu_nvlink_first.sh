#!/bin/bash
# 2 GPUs: NVLink TX/RX bytes of ONE fused-push stage kernel under ncu — the
# first stage-1 launch of rank 0 (the call's first stage waits for no peer, so
# replaying it cannot stall; the peer's waits have a 20 s deadline), against
# the halo plan (slabs x 192 cells x nf x 8 B).  rank 1 runs plain.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export MASTER_ADDR=127.0.0.1 MASTER_PORT=$((29000 + RANDOM % 500)) WORLD_SIZE=2 TS_HYDRO_WAIT_TIMEOUT_MS=60000
M="nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
RANK=0 LOCAL_RANK=0 timeout 600 ncu --metrics $M --clock-control none -k regex:stage_kernel --launch-skip 0 --launch-count 1 --csv \
   python tools/nvlink_bytes.py --steps 2 > gpurun_out/nvlink_first_r0.log 2>&1 &
P0=$!
RANK=1 LOCAL_RANK=1 timeout 600 python tools/nvlink_bytes.py --steps 2 > gpurun_out/nvlink_first_r1.log 2>&1
echo "rank1 rc=$?"
wait $P0; echo "rank0 rc=$?"
grep -E "nvl|gpu__time|dram|^\{" gpurun_out/nvlink_first_r0.log | tail -20
tail -2 gpurun_out/nvlink_first_r1.log
