#!/bin/bash
# K sweep for the latency-bound configs 2 and 3 (the backward / fit plan; forward by its own model)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/small_sweep.txt; : > $out
for K in 0 1 2 3 5 13; do
  for c in 2 3; do
    r=$(NURBS_PLAN_K=$K timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e 2>>gpurun_out/small_sweep.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms %.5f value %.4g plan %s' % (d['ms_per_step'], d['value'], d.get('plan')))" 2>&1)
    echo "cfg$c K=$K $r" | tee -a $out
  done
done
