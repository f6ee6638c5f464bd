#!/bin/bash
# Baseline bench lines (cfg4, cfg5) + one ncu --set full capture (with source) of the cfg4 backward.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-base}
for cfg in 4 5; do timeout 300 python bench.py --config $cfg --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_cfg$cfg.json 2>gpurun_out/bench_${TAG}_cfg$cfg.log; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s ${SKIP:-7} -c 1 -f -o gpurun_out/prof_${TAG} \
    python bench.py --config ${CFG:-4} --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}.log 2>&1
python scripts/sass_hot.py gpurun_out/prof_${TAG}.ncu-rep > gpurun_out/hot_${TAG}.txt 2>&1
tail -3 gpurun_out/bench_${TAG}_cfg4.json gpurun_out/bench_${TAG}_cfg5.json
