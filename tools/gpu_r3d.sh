cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3d
timeout 1200 bash tools/ab_bench.sh "1 4 2" 3 > gpurun_out/r3d/ab.txt 2>&1; cat gpurun_out/r3d/ab.txt
