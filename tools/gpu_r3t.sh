cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3t
o=gpurun_out/r3t
timeout 1500 bash tools/ab_bench.sh "2 5" 2 > $o/ab.txt 2>&1; cat $o/ab.txt
