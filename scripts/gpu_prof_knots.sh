#!/bin/bash
# ncu --set full of the knot-gradient backward (grid kernel mode 3) on config 4, with the
# per-line attribution (exp/grid_p3.cubin = the P = 3 unit of the shipped library)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/kg; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s 3 -c 1 -f -o /tmp/kg python bench.py --knots --steps 3 --warmup 3 > $O/ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches.csv python bench.py --knots --steps 3 --warmup 3 > /dev/null 2>&1
python scripts/sass_hot.py /tmp/kg.ncu-rep > $O/hot.txt 2>&1
MODE=outer python scripts/sass_lines.py /tmp/kg.ncu-rep exp/grid_p3.cubin _ZN2nb17nurbs_grid_kernelILi3ELi3ELb1ELi1ELb0ELb1EEEvNS_6ParamsE . 60 > $O/lines.txt 2>&1
MODE=both python scripts/sass_lines.py /tmp/kg.ncu-rep exp/grid_p3.cubin _ZN2nb17nurbs_grid_kernelILi3ELi3ELb1ELi1ELb0ELb1EEEvNS_6ParamsE . 80 > $O/lines_both.txt 2>&1
