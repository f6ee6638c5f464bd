#!/bin/bash
# Round-end check on the final library: the GPU suite, smoke(), then every bench line and the
# ncu evidence (scripts/gpu_bench_final.sh).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/final
if [ -z "$NO_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
tail -3 gpurun_out/final/pytest_gpu.log
fi
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
tail -2 gpurun_out/final/smoke.log
bash scripts/gpu_bench_final.sh
ls gpurun_out/final
