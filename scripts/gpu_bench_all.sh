#!/bin/bash
# Full bench lines: config 4 default (incl. cpu_baseline + e2e), config 5, config 3 (fit),
# derivatives, knot gradients, paired points, and the reference (oracle) arm.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "default rc=$?"
timeout 600 python bench.py --config 5 --steps 100 --warmup 5 > gpurun_out/bench_cfg5.log 2>&1; echo "cfg5 rc=$?"
timeout 600 python bench.py --config 3 > gpurun_out/bench_cfg3.log 2>&1; echo "cfg3 rc=$?"
timeout 600 python bench.py --derivs --no-cpu-baseline --no-e2e > gpurun_out/bench_derivs.log 2>&1; echo "derivs rc=$?"
timeout 600 python bench.py --knots --no-cpu-baseline --no-e2e > gpurun_out/bench_knots4.log 2>&1; echo "knots4 rc=$?"
timeout 600 python bench.py --knots --config 5 --steps 50 --no-cpu-baseline --no-e2e > gpurun_out/bench_knots5.log 2>&1; echo "knots5 rc=$?"
timeout 600 python bench.py --paired --no-cpu-baseline --no-e2e > gpurun_out/bench_paired.log 2>&1; echo "paired rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo "ref rc=$?"
for f in default cfg5 cfg3 derivs knots4 knots5 paired reference; do echo "== $f"; tail -c 600 gpurun_out/bench_$f.log; echo; done
