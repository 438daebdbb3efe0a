# usage (under gpurun): per-leg and look-back probes of every tools/variants/*.so (via VT_LIB)
for f in tools/variants/*.so; do
  echo "== $f"; VT_LIB=$f python tools/leg_times.py 2>&1 | grep -E "cfg2|cfg5"; VT_LIB=$f python tools/probe.py 2>&1 | grep lookback
done
