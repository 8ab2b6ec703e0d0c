cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 1200 python -m pytest tests/test_gpu_layer.py tests/test_gpu_chain.py tests/test_gpu_multi.py -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/r59_tests.log 2>&1; echo "exit $?" >> gpurun_out/r59_tests.log
tail -n 2 gpurun_out/r59_tests.log
grep -q "exit 0" gpurun_out/r59_tests.log || exit 1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r59_b1.log 2>&1; echo "exit $?" >> gpurun_out/r59_b1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 > gpurun_out/r59_b4.log 2>&1; echo "exit $?" >> gpurun_out/r59_b4.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 > gpurun_out/r59_b2.log 2>&1; echo "exit $?" >> gpurun_out/r59_b2.log
