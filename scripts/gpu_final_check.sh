#!/bin/bash
# Final check of the committed library: the GPU suite, smoke(), the config 4 / 5 bench lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/fc
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fc/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fc/pytest_gpu.log
tail -2 gpurun_out/fc/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fc/smoke.log
tail -2 gpurun_out/fc/smoke.log
timeout 600 python bench.py > gpurun_out/fc/cfg4.jsonl 2> gpurun_out/fc/cfg4.log; echo "cfg4 rc=$?"
timeout 600 python bench.py --config 5 > gpurun_out/fc/cfg5.jsonl 2> gpurun_out/fc/cfg5.log; echo "cfg5 rc=$?"
