#!/bin/bash
# The self-check build (TS_CHECK=1) over the sanitize cases and the GPU suite
# (compute-sanitizer is not available on this pool).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/selfcheck
export TS_HYDRO_LIB=$PWD/paper_2210_06437_b200/libts_hydro_check.so
python tools/sanitize_cases.py > gpurun_out/selfcheck/cases.log 2>&1; echo "cases rc=$?"; cat gpurun_out/selfcheck/cases.log
TS_HYDRO_CHECK_STRICT=1 timeout 2400 python -m pytest tests -q -m gpu -k "not multirank and not two_gpu" > gpurun_out/selfcheck/suite.log 2>&1; echo "suite rc=$?"; tail -5 gpurun_out/selfcheck/suite.log
TS_HYDRO_CHECK_STRICT=1 timeout 900 python -m pytest tests/test_gpu_multirank.py -q -k "one_gpu" > gpurun_out/selfcheck/multirank.log 2>&1; echo "multirank rc=$?"; tail -3 gpurun_out/selfcheck/multirank.log
