#!/bin/bash
# Round-2 bench lines: every config, the shard shapes, the NEXT rows, the reference arm,
# plus the ncu launch lists (cfg4 / cfg5) and one --set full capture of the cfg4 backward.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
out=gpurun_out/bench_r02.jsonl; : > $out; : > gpurun_out/bench_r02.log
run() { echo "### $*" >> gpurun_out/bench_r02.log; timeout 900 python bench.py "$@" >> $out 2>> gpurun_out/bench_r02.log; echo "rc=$? $*" >> gpurun_out/bench_r02.log; }
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
if [ -z "$SKIP_NCU" ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  ncu --set full --clock-control none -k regex:nurbs_grid_kernel -s 7 -c 1 -f -o gpurun_out/prof_r02_cfg4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  ncu --set full --clock-control none -k regex:nurbs_grid_kernel -s 7 -c 1 -f -o gpurun_out/prof_r02_cfg5 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
fi
python - <<'PY'
import json
for l in open("gpurun_out/bench_r02.jsonl"):
    try: d = json.loads(l)
    except Exception: continue
    c = d.get("config", {})
    print(c.get("workload", d.get("metric"))[:5], c.get("shard", "")[:12], d.get("impl", ""), "%.4g" % d["value"], "ms %.4f" % d["ms_per_step"],
          "fwd", d.get("fwd_ms") or d.get("fwd_us"), "bwd", d.get("bwd_ms") or d.get("bwd_us"),
          "frac", (d.get("roofline") or {}).get("frac"), "cpu", (d.get("cpu_baseline") or {}).get("value"), (d.get("cpu_baseline") or {}).get("cores"), "clk", (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"))
PY
