#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s 1 -c 1 -f -o gpurun_out/prof_knots \
    python bench.py --knots --steps 1 --warmup 3 > gpurun_out/ncu_full_knots.log 2>&1
tail -2 gpurun_out/ncu_full_knots.log
