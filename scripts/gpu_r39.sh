cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu --timeout 120 -p no:cacheprovider -k "ar or layernorm or colsum" > gpurun_out/r39_kern.log 2>&1; echo "exit $?" >> gpurun_out/r39_kern.log
for T in 2 4; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $T --master-addr 127.0.0.1 --master-port 2956$T tools/ar_sweep.py > gpurun_out/r39_ar_T$T.json 2> gpurun_out/r39_ar_T$T.err
done
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 800 -p no:cacheprovider -s > gpurun_out/r39_multi.log 2>&1; echo "exit $?" >> gpurun_out/r39_multi.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 > gpurun_out/r39_b4.log 2>&1; echo "exit $?" >> gpurun_out/r39_b4.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 > gpurun_out/r39_b2.log 2>&1; echo "exit $?" >> gpurun_out/r39_b2.log
tail -n 2 gpurun_out/r39_kern.log gpurun_out/r39_multi.log; grep -h '"res"' gpurun_out/r39_ar_T*.json
