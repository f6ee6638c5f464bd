#!/bin/bash
# ncu evidence for profiles/: launch lists of configs 4 / 5 and one --set full capture of the
# forward and backward grid kernels each, summarised ON the box (reports stay in /tmp: too big
# to bring back), plus the per-source-line attribution of the config-4 backward.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/final; mkdir -p $O /tmp/ncu
TAG=${TAG:-r02}
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_cfg4.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_cfg5.csv python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s 6 -c 2 -f -o /tmp/ncu/cfg4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s 6 -c 2 -f -o /tmp/ncu/cfg5 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_summary.py --tag ${TAG}_cfg4 --cfg 4 --launches $O/launches_cfg4.csv --full /tmp/ncu/cfg4.ncu-rep > /dev/null 2>&1
python scripts/ncu_summary.py --tag ${TAG}_cfg5 --cfg 5 --launches $O/launches_cfg5.csv --full /tmp/ncu/cfg5.ncu-rep > /dev/null 2>&1
cp profiles/${TAG}_cfg4_* profiles/${TAG}_cfg5_* profiles/ncu_traffic.json $O/
python scripts/sass_hot.py /tmp/ncu/cfg4.ncu-rep "1, 1, 0, 0" > $O/${TAG}_cfg4_bwd_hot.txt 2>&1
MODE=outer python scripts/sass_lines.py /tmp/ncu/cfg4.ncu-rep exp/grid_p3.cubin _ZN2nb17nurbs_grid_kernelILi3ELi3ELb1ELi1ELb0ELb0EEEvNS_6ParamsE "3, 1, 1" 60 > $O/${TAG}_cfg4_bwd_lines.txt 2>&1
ls -la $O
