# bounds-checked build (-DVT_CHECKS=1) of the round's final kernels over the sanitize workload and all GPU tests;
# compute-sanitizer attempt (refused on this pool so far)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2x
o=gpurun_out/r2x
(timeout 120 compute-sanitizer --tool memcheck python tools/sanitize.py 2>&1 | tail -5) > $o/compute_sanitizer_attempt.txt; echo rc=$? >> $o/compute_sanitizer_attempt.txt
VT_LIB=tools/probes/checked.so python tools/sanitize.py > $o/checked_sanitize.txt 2>&1; echo rc=$? >> $o/checked_sanitize.txt
VT_LIB=tools/probes/checked.so timeout 1800 python -m pytest tests -q -m gpu > $o/checked_pytest_gpu.txt 2>&1; echo rc=$? >> $o/checked_pytest_gpu.txt
tail -3 $o/compute_sanitizer_attempt.txt $o/checked_sanitize.txt $o/checked_pytest_gpu.txt
