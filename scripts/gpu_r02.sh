#!/bin/bash
# Round-2 GPU session: GPU tests (parity log), smoke, and the bench lines of every config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; grep -m1 "model name" /proc/cpuinfo >> gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
NB_PARITY_LOG=gpurun_out/parity_r02.jsonl timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
if [ -z "$SKIP_BENCH" ]; then
  : > gpurun_out/bench_r02.jsonl
  for a in "" "--config 5" "--config 1" "--config 2" "--config 3" \
           "--shard-of 2 --no-cpu-baseline --no-e2e" "--shard-of 4 --no-cpu-baseline --no-e2e" "--shard-of 8 --no-cpu-baseline --no-e2e" \
           "--config 5 --shard-of 2 --no-cpu-baseline --no-e2e" "--config 5 --shard-of 4 --no-cpu-baseline --no-e2e" "--config 5 --shard-of 8 --no-cpu-baseline --no-e2e" \
           "--impl reference" ; do
    echo "### $a" >> gpurun_out/bench_r02.log
    timeout 600 python bench.py $a >> gpurun_out/bench_r02.jsonl 2>> gpurun_out/bench_r02.log
    echo "rc=$? $a" >> gpurun_out/bench_r02.log
  done
  python - <<'PY'
import json
for l in open("gpurun_out/bench_r02.jsonl"):
    try: d = json.loads(l)
    except Exception: continue
    c = d.get("config", {})
    print(c.get("workload", "")[:5], c.get("shard", "")[:12], d.get("impl", ""), "%.4g" % d["value"], "ms", "%.4f" % d["ms_per_step"],
          "fwd", d.get("fwd_ms") or d.get("fwd_us"), "bwd", d.get("bwd_ms") or d.get("bwd_us"),
          "frac", (d.get("roofline") or {}).get("frac"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
PY
fi
