cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r64_b1.log 2>&1; echo "exit $?" >> gpurun_out/r64_b1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r64_b2.log 2>&1; echo "exit $?" >> gpurun_out/r64_b2.log
