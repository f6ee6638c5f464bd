#!/bin/bash
# ncu --set full of the paired-points fwd and bwd kernels (one launch each).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-pts}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nurbs_points_ -s 6 -c 2 -f -o gpurun_out/prof_${TAG} \
    python bench.py --paired --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_full_${TAG}.log
