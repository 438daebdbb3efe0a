cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2e
VT_LIB=tools/variants/traced.so python tools/cfg4_trace.py > gpurun_out/r2e/cfg4_trace.txt 2>&1
VT_LIB=tools/variants/checked.so timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2e/checked_pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/r2e/checked_pytest_gpu.txt
