cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 600 -p no:cacheprovider -s > gpurun_out/r12_multi.log 2>&1; echo "exit $?" >> gpurun_out/r12_multi.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/r12_bench2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --n-sub 4 > gpurun_out/r12_bench2_n4.log 2>&1
timeout 600 python bench.py > gpurun_out/r12_bench1.log 2>&1
