# usage (under gpurun): end-to-end probe of every tools/variants/*.so (via VT_LIB)
for f in tools/variants/*.so; do
  echo "== $f"; VT_LIB=$f python tools/e2e_probe.py 2>&1 | grep -E "e2e|Error"
done
