cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 600 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 500 -p no:cacheprovider -k "2" > gpurun_out/r62_multi.log 2>&1; echo "exit $?" >> gpurun_out/r62_multi.log
for i in 1 2 3 4 5; do
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2958$i bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r62_b2_$i.log 2>&1; echo "exit $?" >> gpurun_out/r62_b2_$i.log
tail -n 1 gpurun_out/r62_b2_$i.log
done
grep -h "stalled" gpurun_out/r62_b2_*.log | head
