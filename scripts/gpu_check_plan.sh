#!/bin/bash
# GPU tests (all) + the default plans at the per-rank shard shapes.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
out=gpurun_out/plan_default.txt; : > $out
for c in 4 5; do for G in 1 2 4 8; do
  r=$(timeout 300 python bench.py --config $c --shard-of $G --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>>gpurun_out/plan_default.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fwd %.4f bwd %.4f plan %s rows %s' % (d['fwd_ms'], d['bwd_ms'], d.get('plan'), d.get('ctrl_rows')))" 2>&1)
  echo "cfg$c G=$G $r" | tee -a $out
done; done
