#!/bin/bash
# Quick GPU iteration: gpu tests (optionally filtered), bench cfg4 + cfg5 kernel-only lines.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 4 5; do
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_q$c.log 2>&1
done
tail -4 gpurun_out/pytest_gpu.log
for c in 4 5; do python - <<PY
import json
l=[x for x in open("gpurun_out/bench_q$c.log") if x.startswith("{")][-1]; d=json.loads(l)
r=d["roofline"]; print("cfg$c", "value %.3g"%d["value"], "ms", round(d["ms_per_step"],4), "fwd", round(r["fwd"]["ms"],4), round(r["fwd"]["frac"],3), "bwd", round(r["bwd"]["ms"],4), round(r["bwd"]["frac"],3))
PY
done
