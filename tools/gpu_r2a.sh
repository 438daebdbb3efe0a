cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2a
timeout 900 python -m pytest tests/test_gpu_runtime.py tests/test_gpu_batch.py tests/test_dropin_headers.py -q -x > gpurun_out/r2a/new_tests.txt 2>&1; echo rc=$? >> gpurun_out/r2a/new_tests.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/r2a/pytest_gpu.txt 2>&1; echo rc=$? >> gpurun_out/r2a/pytest_gpu.txt
timeout 300 python bench.py > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; echo rc=$? >> gpurun_out/r2a/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2a/bench_ref.json 2> gpurun_out/r2a/bench_ref.err
