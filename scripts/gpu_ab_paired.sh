#!/bin/bash
# A/B of the paired-point kernels (bench.py --paired) over experiment libraries
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/ab_paired_${AB_TAG:-x}.txt; : > $out
for rep in 1 2; do for lib in "$@"; do
  r=$(NURBS_B200_LIB_EXPERIMENT=$PWD/$lib timeout 300 python bench.py --paired --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwd %.4f bwd %.4f' % (d['fwd_ms'], d['bwd_ms']))" 2>&1)
  echo "$lib $r" | tee -a $out
done; done
