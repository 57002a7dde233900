#!/bin/bash
# Round-2 evidence run: full GPU suite, smoke, bench (ours + reference), and the
# self-check build over the suite.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/final/suite.log 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/final/suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final/smoke.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo "ref rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench rc=$?"
export TS_HYDRO_LIB=$PWD/paper_2210_06437_b200/libts_hydro_check.so
python tools/sanitize_cases.py > gpurun_out/final/selfcheck_cases.log 2>&1; echo "selfcheck cases rc=$?"; tail -2 gpurun_out/final/selfcheck_cases.log
TS_HYDRO_CHECK_STRICT=1 timeout 2400 python -m pytest tests -q -m gpu -k "not two_gpu and not mismatched_collective" > gpurun_out/final/selfcheck_suite.log 2>&1; echo "selfcheck suite rc=$?"; tail -3 gpurun_out/final/selfcheck_suite.log
