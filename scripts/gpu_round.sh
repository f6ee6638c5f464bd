#!/bin/bash
# One gpurun call: GPU tests + smoke + default bench + ncu (launch list and --set full with source) for a config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash scripts/gpu_check.sh > gpurun_out/check.log 2>&1
TAG=${TAG:-cfg4} CFG=${CFG:-4} bash scripts/gpu_ncu.sh > gpurun_out/ncu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -c 1500 gpurun_out/bench.log
