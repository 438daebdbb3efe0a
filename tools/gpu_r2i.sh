cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2i
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2i/pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/r2i/pytest_gpu.txt
VT_LIB=tools/trace/traced.so python tools/cfg4_trace.py > gpurun_out/r2i/cfg4_trace.txt 2>&1
python tools/cfg4_probe.py > gpurun_out/r2i/cfg4_probe.txt 2>&1
bash tools/ab_bench.sh "2 3" 2 > gpurun_out/r2i/ab.txt 2>&1
for c in 1 4 5; do python bench.py --config $c --no-cpu-baseline --no-e2e --no-rt > gpurun_out/r2i/bench_cfg$c.json 2>/dev/null; done
