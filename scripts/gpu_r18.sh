cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=5000 MERAK_BENCH_TRACE=1 MERAK_BENCH_TRACE_S=60
timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r18_b2.log 2>&1
echo "exit $?" >> gpurun_out/r18_b2.log
