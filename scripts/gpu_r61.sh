cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
for i in 1 2 3 4 5 6 7 8; do
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2957$i bench.py --gpus 2 --no-cpu-baseline --no-extras > gpurun_out/r61_b2_$i.log 2>&1; echo "exit $?" >> gpurun_out/r61_b2_$i.log
tail -n 1 gpurun_out/r61_b2_$i.log
done
grep -h "stalled" gpurun_out/r61_b2_*.log | head
