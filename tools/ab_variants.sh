for f in tools/variants/*.so; do
  cp $f paper_2109_10433_b200/lib/libvtrans_gpu.so
  echo "== $f"; python tools/leg_times.py 2>&1 | grep -E "cfg2|cfg5"; python tools/probe.py 2>&1 | grep lookback
done
