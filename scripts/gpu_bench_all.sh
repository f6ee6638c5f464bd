#!/bin/bash
# Full bench lines (config 4 default incl. cpu_baseline + e2e, config 5, reference arm) and the config-5 ncu capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "default rc=$?"
timeout 600 python bench.py --config 5 --steps 100 --warmup 5 > gpurun_out/bench_cfg5.log 2>&1; echo "cfg5 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
TAG=cfg5 CFG=5 bash scripts/gpu_ncu.sh > /dev/null 2>&1; echo "ncu cfg5 rc=$?"
tail -c 2500 gpurun_out/bench_default.log; echo; tail -c 1500 gpurun_out/bench_cfg5.log; echo; tail -c 800 gpurun_out/bench_reference.log
