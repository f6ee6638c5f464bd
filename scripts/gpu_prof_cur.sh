cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pc
NURBS_B200_LIB_EXPERIMENT=$PWD/exp/lib_cur.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:nurbs_grid_kernel -s 7 -c 1 -f -o /tmp/pc python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/sass_hot.py /tmp/pc.ncu-rep > gpurun_out/pc/hot.txt 2>&1
MODE=outer python scripts/sass_lines.py /tmp/pc.ncu-rep exp/cur_p3.cubin _ZN2nb17nurbs_grid_kernelILi3ELi3ELb1ELi1ELb0ELb0EEEvNS_6ParamsE . 50 > gpurun_out/pc/lines.txt 2>&1
MODE=both python scripts/sass_lines.py /tmp/pc.ncu-rep exp/cur_p3.cubin _ZN2nb17nurbs_grid_kernelILi3ELi3ELb1ELi1ELb0ELb0EEEvNS_6ParamsE . 80 > gpurun_out/pc/lines_both.txt 2>&1
