#!/bin/bash
# Plan sweep: per-rank shard shapes (cfg4 B = 4096/G, cfg5 windowed u-slabs) with the row-block
# size K forced (NURBS_PLAN_K backward, NURBS_PLAN_KF forward); fwd/bwd ms per setting.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/plan_sweep.txt; : > $out
one() {  # cfg G K
  r=$(NURBS_PLAN_K=$3 NURBS_PLAN_KF=$3 timeout 300 python bench.py --config $1 --shard-of $2 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>>gpurun_out/plan_sweep.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwd %.4f bwd %.4f plan %s rows %s' % (d['fwd_ms'], d['bwd_ms'], d.get('plan'), d.get('ctrl_rows')))" 2>&1)
  echo "cfg$1 G=$2 K=$3 $r" | tee -a $out
}
for G in 1 2 4 8; do for K in 0 13 7 5 4 3 2 1; do one 4 $G $K; done; done
for G in 1 2 4 8; do for K in 0 13 7 4 2 1; do one 5 $G $K; done; done
