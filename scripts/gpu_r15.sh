cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=5000 MERAK_BENCH_TRACE=1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r15_b2.log 2>&1
echo "exit $?" >> gpurun_out/r15_b2.log
