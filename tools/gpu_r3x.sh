cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3x
o=gpurun_out/r3x
timeout 1500 python -m pytest tests -q -m gpu -x > $o/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 $o/pytest_gpu.log
for c in 2 3 5; do python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg$c', d['ms_per_step'], d['roofline']['frac'])"; done > $o/bench.txt; cat $o/bench.txt
