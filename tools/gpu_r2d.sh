# bounds-checked build over the GPU tests + sanitize workload; cfg4 probe; bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2d
VT_LIB=tools/variants/checked.so python tools/sanitize.py > gpurun_out/r2d/checked_sanitize.txt 2>&1; echo rc=$? >> gpurun_out/r2d/checked_sanitize.txt
VT_LIB=tools/variants/checked.so timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/r2d/checked_pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/r2d/checked_pytest_gpu.txt
python tools/cfg4_probe.py > gpurun_out/r2d/cfg4_probe.txt 2>&1
for c in 1 2 3 4; do python bench.py --config $c --no-cpu-baseline --no-e2e --no-rt > gpurun_out/r2d/bench_cfg$c.json 2>/dev/null; done
