#!/bin/bash
# ncu launch list of the knot-gradient call (config $CFG) for the experiment library $1
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
v=$(basename $1 .so)
NURBS_B200_LIB_EXPERIMENT=$PWD/$1 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/kl_${v}_cfg${CFG:-4}.csv python bench.py --knots --config ${CFG:-4} --steps 3 --warmup 3 > /dev/null 2>&1
