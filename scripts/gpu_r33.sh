cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 800 -p no:cacheprovider -s > gpurun_out/r33_multi.log 2>&1; echo "exit $?" >> gpurun_out/r33_multi.log
timeout 600 python bench.py > gpurun_out/r33_b1.log 2>&1; echo "exit $?" >> gpurun_out/r33_b1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 > gpurun_out/r33_b2.log 2>&1; echo "exit $?" >> gpurun_out/r33_b2.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 > gpurun_out/r33_b4.log 2>&1; echo "exit $?" >> gpurun_out/r33_b4.log
tail -n 3 gpurun_out/r33_multi.log
