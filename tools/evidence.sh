# usage (under gpurun): bash tools/evidence.sh <tag>
# Round evidence: smoke, all GPU tests, bench lines for every config, the
# reference arm, and ncu (launch list + one --set full capture) for cfg2 / cfg3.
tag=${1:-r1g}
mkdir -p gpurun_out/$tag
o=gpurun_out/$tag
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $o/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -q -m gpu > $o/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 $o/pytest_gpu.log
python bench.py > $o/bench_cfg2_default.json 2> $o/bench_cfg2_default.err; echo bench_rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_cfg2_reference_arm.json 2> $o/bench_ref.err; echo ref_rc=$?
for c in 1 3 4 5; do
  python bench.py --config $c --no-cpu-baseline > $o/bench_cfg$c.json 2> $o/bench_cfg$c.err; echo bench_cfg${c}_rc=$?
done
for c in 2 3; do
  k=$([ $c = 3 ] && echo utf16_transcode || echo utf8_transcode)
  bash tools/profile.sh ${tag}_cfg$c $k --steps 2 --warmup 3 --config $c --no-cpu-baseline --no-e2e > /dev/null 2>&1
  mv gpurun_out/${tag}_cfg$c* $o/ 2>/dev/null
  python tools/ncu_summary.py $o/${tag}_cfg$c.ncu-rep > $o/${tag}_cfg${c}_ncu_full_summary.txt 2>&1
  python tools/ncu_lines.py $o/${tag}_cfg$c.ncu-rep 60 > $o/${tag}_cfg${c}_source_lines.txt 2>&1
done
echo done
