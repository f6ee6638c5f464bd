#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck on scripts/sanitize_cases.py (every case);
# logs under gpurun_out/sanitize_<tool>.log (summaries copied to profiles/ by hand)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no --padding 64"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
