#!/bin/bash
# Same-box A/B of the built library variants (bench only) + e2e chunk sweep.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu.py tests/test_harness.py -x -q -k "sedov_4096 or random_state or harness or timing_hook or config3" > gpurun_out/t_ab2.log 2>&1; echo "tests rc=$?"
rm -f gpurun_out/variants.log
for rep in 1 2; do
for lib in ${LIBS:-paper_2210_06437_b200/libts_hydro*.so}; do
  echo "== $(basename $lib)" >> gpurun_out/variants.log
  TS_HYDRO_LIB=$PWD/$lib timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e $BENCH_ARGS >> gpurun_out/variants.log 2>&1
done
done
python tools/variants.py gpurun_out/variants.log
if [ -n "$E2E" ]; then
rm -f gpurun_out/e2e.log
for ch in 4 8 16 32; do
  echo "== chunks $ch" >> gpurun_out/e2e.log
  TS_HYDRO_XFER_CHUNKS=$ch timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/e2e.log 2>&1
done
echo "== chunks 8 nogate" >> gpurun_out/e2e.log
TS_HYDRO_H2D_GATE=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/e2e.log 2>&1
python - <<'PY'
import json
cur=None
for line in open("gpurun_out/e2e.log"):
    if line.startswith("=="): cur=line.strip(); continue
    if line.startswith("{"):
        d=json.loads(line); print(cur, "e2e %.3f G  sync %.3f G" % (d["e2e"]["value"]/1e9, d["e2e"]["sync_value"]/1e9))
PY
fi
