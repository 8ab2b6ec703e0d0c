cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/r6_topo.log 2>&1
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -s > gpurun_out/r6_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r6_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r6_bench1.log 2>&1; echo "bench exit $?" >> gpurun_out/r6_bench1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/r6_bench2.log 2>&1; echo "bench2 exit $?" >> gpurun_out/r6_bench2.log
