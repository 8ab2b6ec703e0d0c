cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/g_tests.log 2>&1; echo "exit $?" >> gpurun_out/g_tests.log
timeout 600 python bench.py > gpurun_out/g_b1.log 2>&1; echo "exit $?" >> gpurun_out/g_b1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 > gpurun_out/g_b2.log 2>&1; echo "exit $?" >> gpurun_out/g_b2.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 > gpurun_out/g_b4.log 2>&1; echo "exit $?" >> gpurun_out/g_b4.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --impl reference --steps 3 --warmup 1 > gpurun_out/g_ref4.log 2>&1; echo "exit $?" >> gpurun_out/g_ref4.log
tail -n 2 gpurun_out/g_tests.log; tail -n 1 gpurun_out/g_ref4.log
