cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29552 tools/ar_sweep.py > gpurun_out/r38_ar_T2.json 2> gpurun_out/r38_ar_T2.err
cat gpurun_out/r38_ar_T2.json
