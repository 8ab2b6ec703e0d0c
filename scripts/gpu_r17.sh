cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=5000
timeout 180 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 tools/chain_debug.py > gpurun_out/r17_dbg.log 2>&1
echo "exit $?" >> gpurun_out/r17_dbg.log
