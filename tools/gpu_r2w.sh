cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2w
for f in tools/variants/*.so; do echo $f; VT_LIB=$f python tools/validate_times.py; VT_LIB=$f python tools/validate_times.py; done > gpurun_out/r2w/validate.txt 2>&1
cat gpurun_out/r2w/validate.txt
timeout 600 python -m pytest tests -q -m gpu -x -k "not acceptance and not fuzz and not full_size and not round_trip" > gpurun_out/r2w/pytest.log 2>&1; tail -2 gpurun_out/r2w/pytest.log
