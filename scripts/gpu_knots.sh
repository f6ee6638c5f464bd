#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_knots.py -x -q > gpurun_out/pytest_knots.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_knots.log
tail -30 gpurun_out/pytest_knots.log
