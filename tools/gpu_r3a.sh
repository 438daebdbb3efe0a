cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3a
o=gpurun_out/r3a
timeout 900 python -m pytest tests -q -m gpu -x -k "not acceptance and not fuzz" > $o/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -5 $o/pytest_gpu.log
python tools/ascii_probe.py > $o/ascii_probe.txt 2>&1; cat $o/ascii_probe.txt
timeout 1200 bash tools/ab_bench.sh "2 3 5 1" 2 > $o/ab.txt 2>&1; cat $o/ab.txt
