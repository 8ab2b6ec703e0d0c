cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=5000 MERAK_BENCH_TRACE=1
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 500 -p no:cacheprovider -s > gpurun_out/r16_multi.log 2>&1; echo "exit $?" >> gpurun_out/r16_multi.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r16_b2.log 2>&1
echo "exit $?" >> gpurun_out/r16_b2.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --no-cpu-baseline --layers 1 > gpurun_out/r16_b2_L1.log 2>&1
