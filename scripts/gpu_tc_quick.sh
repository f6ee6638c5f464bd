cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tensor_core or config2 or config4_small" > gpurun_out/tc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/tc_pytest.log
tail -30 gpurun_out/tc_pytest.log
for e in "NURBS_TC=1" "NURBS_TC=0"; do
  env $e timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', 'fwd %.4f bwd %.4f' % (d['fwd_ms'], d['bwd_ms']))"
done
