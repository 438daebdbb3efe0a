cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r3z
o=gpurun_out/r3z
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 > $o/torchrun_n1.json 2> $o/torchrun_n1.err; echo torchrun_rc=$?; tail -c 600 $o/torchrun_n1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > $o/torchrun_ref_n1.json 2> $o/torchrun_ref_n1.err; echo ref_rc=$?; tail -c 400 $o/torchrun_ref_n1.json
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 > $o/gpus2.json 2> $o/gpus2.err; echo gpus2_rc=$?; tail -3 $o/gpus2.err | cut -c1-300
