#!/bin/bash
# ncu --set full (with source) of the paired kernels matching KRE for the experiment library $1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
lib=$1; v=$(basename $lib .so)
NURBS_B200_LIB_EXPERIMENT=$PWD/$lib timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE:-points_bwd} -s ${SKIP:-3} -c 1 -f -o gpurun_out/prof_${v} \
    python bench.py --paired --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${v}.log 2>&1
tail -2 gpurun_out/ncu_${v}.log
