mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -x -q -m "gpu and not slow" > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -30 gpurun_out/pytest_gpu.log
for c in ${BENCH_CFGS:-2}; do
timeout 300 python bench.py --steps 10 --warmup 3 --config $c $BENCH_ARGS > gpurun_out/bench_cfg$c.log 2>&1; echo bench_rc=$?
tail -2 gpurun_out/bench_cfg$c.log
done
