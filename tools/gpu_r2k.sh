cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2k
o=gpurun_out/r2k
timeout 1200 python -m pytest tests -q -m gpu -x > $o/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $o/pytest_gpu.log
bash tools/ab_bench.sh "3 5" 2 > $o/ab.txt 2>&1; cat $o/ab.txt
