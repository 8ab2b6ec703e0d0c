cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
for cc in 0 296 148 74; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$((cc % 7)) bench.py --gpus 4 --no-cpu-baseline --comm-ctas $cc --steps 10 > gpurun_out/r45_b4_cc$cc.log 2>&1
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$((cc % 7)) bench.py --gpus 2 --no-cpu-baseline --comm-ctas $cc --steps 10 > gpurun_out/r45_b2_cc$cc.log 2>&1
done
