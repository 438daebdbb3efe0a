cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3p
o=gpurun_out/r3p
timeout 900 python -m pytest tests -q -m gpu -x -k "not acceptance and not fuzz" > $o/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $o/pytest_gpu.log
timeout 1500 bash tools/ab_bench.sh "2 3 5 1 4" 2 > $o/ab.txt 2>&1; cat $o/ab.txt
