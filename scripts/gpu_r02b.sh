#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
NB_PARITY_LOG=gpurun_out/parity_r02.jsonl timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/bench_r02b.jsonl
for a in "--no-cpu-baseline --no-e2e" "--tc --no-cpu-baseline --no-e2e" ; do
  timeout 600 python bench.py $a >> gpurun_out/bench_r02b.jsonl 2>> gpurun_out/bench_r02b.log
done
NB_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --no-cpu-baseline --steps 20 >> gpurun_out/bench_r02b.jsonl 2>> gpurun_out/bench_r02b.log
NB_BENCH_SHARE_GPU=1 timeout 600 python bench.py --gpus 2 --config 5 --no-cpu-baseline --no-e2e --steps 20 >> gpurun_out/bench_r02b.jsonl 2>> gpurun_out/bench_r02b.log
python - <<'PY'
import json
for l in open("gpurun_out/bench_r02b.jsonl"):
    try: d = json.loads(l)
    except Exception: continue
    print(d["n_gpus"], d["config"]["global_batch"], d["config"]["points_per_step"], d["config"]["parallelism"], d.get("bwd_path"), "%.4g" % d["value"], d.get("fwd_ms"), d.get("bwd_ms"), (d.get("tc_bwd") or {}).get("ms"), d.get("rank0_units"))
PY
tail -5 gpurun_out/bench_r02b.log
