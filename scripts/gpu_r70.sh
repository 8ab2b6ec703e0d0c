cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000 MERAK_DEBUG_TRACE=1
for i in $(seq 1 18); do
timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29600+i)) bench.py --gpus 2 --no-cpu-baseline --no-extras --steps 40 > gpurun_out/r70_b2_$i.log 2>&1; echo "exit $?" >> gpurun_out/r70_b2_$i.log
tail -n 1 gpurun_out/r70_b2_$i.log
if grep -q "stalled\|ETIMEOUT" gpurun_out/r70_b2_$i.log; then grep -h "stalled\|ETIMEOUT\|device:" gpurun_out/r70_b2_$i.log | head -12; break; fi
done
