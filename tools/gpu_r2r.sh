cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2r
o=gpurun_out/r2r
timeout 1200 bash tools/ab_bench.sh "2 5" 2 > $o/ab.txt 2>&1; cat $o/ab.txt
VT_LIB=tools/probes/probe.so python tools/probe.py 2 > $o/probe.txt 2>&1
VT_LIB=tools/probes/probe.so python tools/probe.py 3 >> $o/probe.txt 2>&1; cat $o/probe.txt
VT_LIB=tools/probes/phases.so python tools/phases.py 2 3 5 > $o/phases.txt 2>&1; cat $o/phases.txt
