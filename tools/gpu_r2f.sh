cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2f
VT_LIB=tools/variants/traced.so python tools/cfg4_trace.py > gpurun_out/r2f/cfg4_trace.txt 2>&1
python tools/cfg4_probe.py > gpurun_out/r2f/cfg4_probe.txt 2>&1
for c in 2 3 4 1; do python bench.py --config $c --no-cpu-baseline --no-e2e --no-rt > gpurun_out/r2f/bench_cfg$c.json 2>/dev/null; done
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2f/pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/r2f/pytest_gpu.txt
