cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2l
for c in 3 2; do
  k=$([ $c = 3 ] && echo utf16_transcode || echo utf8_transcode)
  bash tools/profile.sh r2l_cfg$c $k --steps 2 --warmup 3 --config $c --no-cpu-baseline --no-e2e > /dev/null 2>&1
  mv gpurun_out/r2l_cfg$c* gpurun_out/r2l/ 2>/dev/null
  python tools/ncu_summary.py gpurun_out/r2l/r2l_cfg$c.ncu-rep > gpurun_out/r2l/r2l_cfg${c}_ncu_full_summary.txt 2>&1
  python tools/ncu_lines.py gpurun_out/r2l/r2l_cfg$c.ncu-rep 70 > gpurun_out/r2l/r2l_cfg${c}_source_lines.txt 2>&1
done
cat gpurun_out/r2l/r2l_cfg3_ncu_full_summary.txt
