cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r4a
o=gpurun_out/r4a
timeout 900 python -m pytest tests -q -m gpu -x -k "not acceptance and not fuzz" > $o/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $o/pytest_gpu.log
timeout 1500 bash tools/ab_bench.sh "2 5 4" 2 > $o/ab.txt 2>&1; cat $o/ab.txt
for f in tools/variants/*.so; do echo "$(basename $f): $(VT_LIB=$f python tools/leg_times.py 2>&1 | tail -4 | tr '\n' ' ')"; done > $o/legs.txt 2>&1; cat $o/legs.txt
