cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in 16 32 64 128 256 512; do
  r=$(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-chunk $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4g %.3f' % (d['e2e']['value'], d['e2e']['ms_per_step']))")
  echo "chunk $c e2e $r" | tee -a gpurun_out/e2e_sweep.txt
done
