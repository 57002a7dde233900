#!/bin/bash
# Same-box: N=1 timeline, N replicas timeline, N-rank timelines (fused push, copy engine), bench lines.
N=$(nvidia-smi -L | wc -l)
S=${STEPS:-20}
tl() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $1 tools/timeline.py --quiet --steps $S ${@:2} 2>&1 | grep -E "^rank|summary"; }
echo "== n1"; timeout 300 python tools/timeline.py --quiet --steps $S | grep -E "^rank|summary"
echo "== replicas"; tl 29821 --replicas
for lib in paper_2210_06437_b200/libts_hydro*.so; do
  echo "== $(basename $lib)"; TS_HYDRO_LIB=$lib tl 29822
done
echo "== ce"; TS_HYDRO_HALO=ce tl 29823
if [ -f paper_2210_06437_b200/libts_hydro_nosync.so ]; then
  echo "== nosync natural order"; TS_EXP_NATURAL=1 TS_HYDRO_LIB=paper_2210_06437_b200/libts_hydro_nosync.so tl 29824
fi
