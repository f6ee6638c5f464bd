#!/bin/bash
# One ncu --set full capture (with source) of the fwd and bwd grid kernels for config $CFG.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-x}; CFG=${CFG:-4}
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-nurbs_grid_kernel} -s ${SKIP:-6} -c ${COUNT:-2} -f -o gpurun_out/prof_${TAG} \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_full_${TAG}.log
