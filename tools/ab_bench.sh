# usage (under gpurun, after tools/build_variants.sh): bash tools/ab_bench.sh "<configs>" [rounds]
# Alternates the variant libraries round-robin (loaded through VT_LIB; the
# in-tree product library is never overwritten) and prints ms/step per config.
cfgs=${1:-"2 3"}; rounds=${2:-2}
for r in $(seq $rounds); do
for f in tools/variants/*.so; do
  for c in $cfgs; do
    ms=$(VT_LIB=$f python bench.py --steps 10 --warmup 3 --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'])")
    echo "round $r $(basename $f .so) cfg$c ms/frac: $ms"
  done
done
done
