cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=5000
for n in 1 2; do
NSUB=$n timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$n tools/timeline.py > gpurun_out/r19_tl_n$n.log 2>&1
done
