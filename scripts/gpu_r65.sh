cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r65_b2.log 2>&1; echo "exit $?" >> gpurun_out/r65_b2.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r65_b4.log 2>&1; echo "exit $?" >> gpurun_out/r65_b4.log
timeout 300 python bench.py --no-cpu-baseline --steps 6 > gpurun_out/r65_b1.log 2>&1; echo "exit $?" >> gpurun_out/r65_b1.log
