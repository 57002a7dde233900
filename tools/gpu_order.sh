#!/bin/bash
# Sub-grid numbering A/B: Morton vs row-major (device-resident value and the pipelined e2e).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/order
timeout 300 python -m pytest tests/test_gpu.py -q -k "row_ordered or pipelined" > gpurun_out/order/t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/order/t.log
for rep in 1 2; do
for o in morton row; do
  timeout 300 python bench.py --order $o --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/order/sedov_${o}_$rep.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/order/sedov_${o}_$rep.json')); print('sedov $o', round(d['value']/1e9,3), 'e2e', round(d['e2e']['value']/1e9,3))"
done
done
for o in morton row; do
  timeout 300 python bench.py --order $o --workload polytrope --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/order/poly_${o}.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/order/poly_${o}.json')); print('polytrope $o', round(d['value']/1e9,3))"
done
