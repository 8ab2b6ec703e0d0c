cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=3000
for L in 1 2; do
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2951$L bench.py --gpus 2 --steps 2 --warmup 1 --layers $L --no-extras --no-cpu-baseline > gpurun_out/r14_L$L.log 2>&1
echo "L$L exit $?" >> gpurun_out/r14_L$L.log
done
