cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3q
o=gpurun_out/r3q
timeout 1500 bash tools/ab_bench.sh "2 3" 2 > $o/ab.txt 2>&1; cat $o/ab.txt
