cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3m
o=gpurun_out/r3m
for k in 1 2 3 4; do for c in 2 3; do
  ms=$(VT_OCC_CAP=$k python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])")
  echo "CTAs/SM<=$k cfg$c ms/frac: $ms"
done; done > $o/occ_cap.txt 2>&1; cat $o/occ_cap.txt
