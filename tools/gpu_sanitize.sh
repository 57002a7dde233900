#!/bin/bash
# compute-sanitizer over the synchronisation protocols (tools/sanitize_cases.py) and smoke.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sanitizer
python tools/sanitize_cases.py > gpurun_out/sanitizer/plain.log 2>&1; echo "plain rc=$?"
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$?"
  tail -3 gpurun_out/sanitizer/$tool.log
done
timeout 600 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer/memcheck_smoke.log 2>&1; echo "smoke memcheck rc=$?"
tail -2 gpurun_out/sanitizer/memcheck_smoke.log
