#!/bin/bash
# Round-end evidence: every bench line (configs 1-5, per-rank shard shapes, tcgen05 side path,
# NEXT rows, reference arm, a 2-rank plumbing run), ncu launch lists of configs 4/5 and one
# `--set full` capture of each grid kernel (cfg4 fwd+bwd, cfg5 fwd+bwd).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/final
O=gpurun_out/final
out=$O/bench.jsonl; : > $out; : > $O/bench.log
run() { echo "### $*" >> $O/bench.log; timeout 900 python bench.py "$@" >> $out 2>> $O/bench.log; echo "rc=$? $*" >> $O/bench.log; }
run
run --config 5
run --config 1
run --config 2
run --config 3
for g in 2 4 8; do run --shard-of $g --no-cpu-baseline --no-e2e; run --config 5 --shard-of $g --no-cpu-baseline --no-e2e; done
run --tc --no-cpu-baseline --no-e2e
run --derivs
run --knots
run --knots --config 5
run --paired
run --impl reference
run --impl reference --config 5
NB_BENCH_SHARE_GPU=1 run --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
NB_BENCH_SHARE_GPU=1 run --config 5 --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e
if [ -z "$SKIP_NCU" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_cfg5.csv python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  [ -n "$FULL" ] && ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s 6 -c 2 -f -o $O/prof_cfg4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  [ -n "$FULL" ] && ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s 6 -c 2 -f -o $O/prof_cfg5 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
fi
