#!/bin/bash
# A/B of the knot-gradient backward (bench.py --knots, configs 4 and 5) over experiment libraries
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/ab_knots_${AB_TAG:-x}.txt; : > $out
for rep in 1 2; do for lib in "$@"; do for cfg in 4 5; do
  r=$(NURBS_B200_LIB_EXPERIMENT=$PWD/$lib timeout 300 python bench.py --knots --config $cfg --steps 50 --warmup 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms %.4f frac %.3f' % (d['ms_per_step'], d['roofline']['frac']))" 2>&1)
  echo "$lib cfg$cfg $r" | tee -a $out
done; done; done
