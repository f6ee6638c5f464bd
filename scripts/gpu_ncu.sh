#!/bin/bash
# ncu: launch list of a short bench run + one --set full capture of the fwd and bwd kernels.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-cfg4}
CFG=${CFG:-4}
ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s 6 -c 2 -f -o gpurun_out/prof_${TAG} \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}.log
