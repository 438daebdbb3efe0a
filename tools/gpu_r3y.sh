cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3y
o=gpurun_out/r3y
timeout 1500 bash tools/ab_bench.sh "2 3 5" 3 > $o/ab.txt 2>&1; cat $o/ab.txt
