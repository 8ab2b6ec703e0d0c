cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
for KB in 160 192; do
MERAK_GEMM_SMEM_KB=$KB timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953${KB:0:1} bench.py --gpus 4 --no-cpu-baseline --no-extras > gpurun_out/r67_b4_$KB.log 2>&1; echo "exit $?" >> gpurun_out/r67_b4_$KB.log
MERAK_GEMM_SMEM_KB=$KB timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954${KB:0:1} bench.py --gpus 2 --no-cpu-baseline --no-extras > gpurun_out/r67_b2_$KB.log 2>&1; echo "exit $?" >> gpurun_out/r67_b2_$KB.log
done
for KB in 160 192; do
MERAK_GEMM_SMEM_KB=$KB timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2955${KB:0:1} bench.py --gpus 4 --no-cpu-baseline --no-extras > gpurun_out/r67_b4b_$KB.log 2>&1; echo "exit $?" >> gpurun_out/r67_b4b_$KB.log
done
