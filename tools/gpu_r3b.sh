cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3b
timeout 900 python -m pytest tests -q -m gpu -x -k "not acceptance and not fuzz" > gpurun_out/r3b/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -5 gpurun_out/r3b/pytest_gpu.log
