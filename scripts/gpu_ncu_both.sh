cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
TAG=cfg4v2 CFG=4 bash scripts/gpu_ncu.sh
TAG=cfg5v2 CFG=5 bash scripts/gpu_ncu.sh
ls -la gpurun_out
