cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2u
for c in 2 3; do
  k=$([ $c = 3 ] && echo utf16_transcode || echo utf8_transcode)
  bash tools/profile.sh r2u_cfg$c $k --steps 2 --warmup 3 --config $c --no-cpu-baseline --no-e2e > /dev/null 2>&1
  mv gpurun_out/r2u_cfg$c* gpurun_out/r2u/ 2>/dev/null
  python tools/ncu_summary.py gpurun_out/r2u/r2u_cfg$c.ncu-rep > gpurun_out/r2u/r2u_cfg${c}_ncu_full_summary.txt 2>&1
done
cat gpurun_out/r2u/r2u_cfg2_ncu_full_summary.txt | tail -3
