cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s
timeout 1500 python -m pytest tests -q -m gpu -x -k "config or full_size" > gpurun_out/r2s/pytest_cfg.log 2>&1; echo rc=$?; tail -5 gpurun_out/r2s/pytest_cfg.log
