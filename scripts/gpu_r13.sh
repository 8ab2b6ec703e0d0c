cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -x > gpurun_out/r13_tests.log 2>&1; echo "exit $?" >> gpurun_out/r13_tests.log
timeout 600 python bench.py > gpurun_out/r13_bench1.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/r13_bench2.log 2>&1
