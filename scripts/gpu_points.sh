#!/bin/bash
# One gpurun call for the paired-points path: build, its GPU tests, a bench line, ncu list.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_points.py -x -q > gpurun_out/pytest_points.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_points.log
timeout 600 python bench.py --paired --steps 20 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_paired.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_paired.csv \
    python bench.py --paired --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_paired.log 2>&1
tail -15 gpurun_out/pytest_points.log; tail -c 2500 gpurun_out/bench_paired.log
