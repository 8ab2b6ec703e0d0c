cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000 MERAK_BENCH_TRACE=1 MERAK_BENCH_TRACE_S=150
for i in 1 2 3; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$i bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r50_b4_$i.log 2>&1; echo "exit $?" >> gpurun_out/r50_b4_$i.log
done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r50_b1.log 2>&1; echo "exit $?" >> gpurun_out/r50_b1.log
for i in 1 2 3; do tail -n 1 gpurun_out/r50_b4_$i.log; done
