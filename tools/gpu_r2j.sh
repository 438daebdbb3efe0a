cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2j
bash tools/ab_bench.sh "2 3" 3 > gpurun_out/r2j/ab.txt 2>&1
VT_LIB=tools/trace/traced.so python tools/cfg4_trace.py > gpurun_out/r2j/cfg4_trace.txt 2>&1
python tools/cfg4_probe.py > gpurun_out/r2j/cfg4_probe.txt 2>&1
python bench.py --no-cpu-baseline --no-rt > gpurun_out/r2j/bench_cfg2_e2e.json 2>/dev/null
python bench.py --config 3 --no-cpu-baseline --no-rt > gpurun_out/r2j/bench_cfg3_e2e.json 2>/dev/null
