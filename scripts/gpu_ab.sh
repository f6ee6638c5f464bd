#!/bin/bash
# A/B: bench kernel-only lines of libraries given as arguments (NURBS_B200_LIB_EXPERIMENT), interleaved
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/ab_${AB_TAG:-x}.txt; : > $out
for rep in 1 2; do
 for lib in "$@"; do
  for cfg in ${AB_CONFIGS:-4 5}; do
    r=$(NURBS_B200_LIB_EXPERIMENT=$lib timeout 300 python bench.py --config $cfg --steps 100 --warmup 10 --no-cpu-baseline --no-e2e ${AB_ARGS} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwd %.4f bwd %.4f' % (d['fwd_ms'], d['bwd_ms']))" 2>&1)
    echo "$lib cfg$cfg $r" | tee -a $out
  done
 done
done
