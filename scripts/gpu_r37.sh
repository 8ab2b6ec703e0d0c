cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
for T in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $T --master-addr 127.0.0.1 --master-port 2955$T tools/ar_sweep.py > gpurun_out/r37_ar_T$T.json 2> gpurun_out/r37_ar_T$T.err
done
MERAK_AR_TWO_SHOT=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29559 tools/ar_sweep.py > gpurun_out/r37_ar_T4_oneshot.json 2> gpurun_out/r37_ar_T4_oneshot.err
cat gpurun_out/r37_ar_*.json
