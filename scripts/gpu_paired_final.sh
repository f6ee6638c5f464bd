#!/bin/bash
# GPU tests, the paired-points bench line (with cpu_baseline and e2e), its ncu launch list and
# one --set full capture of the paired kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pts
O=gpurun_out/pts
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 900 python bench.py --paired > $O/bench_paired.jsonl 2> $O/bench_paired.log; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_paired.csv python bench.py --paired --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:nurbs_points_ -s 6 -c 3 -f -o $O/prof_paired python bench.py --paired --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls $O
