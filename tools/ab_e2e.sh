for f in tools/variants/*.so; do
  cp $f paper_2109_10433_b200/lib/libvtrans_gpu.so
  echo "== $f"; python tools/e2e_probe.py 2>&1 | grep -E "e2e|Error"
done
