#!/bin/bash
# ncu --set full (with source) of the cfg4 backward for each experiment library given as an argument
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for lib in "$@"; do
  v=$(basename $lib .so)
  NURBS_B200_LIB_EXPERIMENT=$PWD/$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s ${SKIP:-7} -c 1 -f -o gpurun_out/prof_${v} \
    python bench.py --config ${CFG:-4} --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${v}.log 2>&1
done
