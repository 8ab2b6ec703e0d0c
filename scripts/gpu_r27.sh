cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000 MERAK_BENCH_TRACE=1
nvidia-smi topo -m > gpurun_out/r27_topo.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 800 -p no:cacheprovider -s > gpurun_out/r27_multi.log 2>&1; echo "exit $?" >> gpurun_out/r27_multi.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 > gpurun_out/r27_b4.log 2>&1; echo "exit $?" >> gpurun_out/r27_b4.log
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 tools/timeline.py > gpurun_out/r27_tl4.log 2>&1
