cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
for T in 2 4; do
for P in 0 1; do
MERAK_AR_PDL=$P timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $T --master-addr 127.0.0.1 --master-port 296$T$P tools/ar_sweep.py > gpurun_out/r63_ar_T${T}_pdl$P.json 2> gpurun_out/r63_ar_T${T}_pdl$P.err
done; done
MERAK_AR_PDL=1 timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 800 -p no:cacheprovider > gpurun_out/r63_multi.log 2>&1; echo "exit $?" >> gpurun_out/r63_multi.log
for P in 0 1; do
MERAK_AR_PDL=$P timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$P bench.py --gpus 4 --no-cpu-baseline > gpurun_out/r63_b4_pdl$P.log 2>&1; echo "exit $?" >> gpurun_out/r63_b4_pdl$P.log
MERAK_AR_PDL=$P timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$P bench.py --gpus 2 --no-cpu-baseline > gpurun_out/r63_b2_pdl$P.log 2>&1; echo "exit $?" >> gpurun_out/r63_b2_pdl$P.log
done
grep -h '"res"' gpurun_out/r63_ar_*.json; tail -n 2 gpurun_out/r63_multi.log
