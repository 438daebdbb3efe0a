cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2b
./tools/pipe_probe_bin > gpurun_out/r2b/pipe_probe.txt 2>&1
ncu --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_alu_cycles_active.sum,sm__pipe_fma_cycles_active.sum,sm__pipe_fmaheavy_cycles_active.sum,smsp__inst_executed.sum,sm__cycles_elapsed.max --csv ./tools/pipe_probe_bin > gpurun_out/r2b/pipe_probe_ncu.csv 2>&1
bash tools/ab_bench.sh "2 3" 2 > gpurun_out/r2b/ab.txt 2>&1
