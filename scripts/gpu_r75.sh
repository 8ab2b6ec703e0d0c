cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/r75_tests.log 2>&1; echo "exit $?" >> gpurun_out/r75_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r75_smoke.log 2>&1; echo "exit $?" >> gpurun_out/r75_smoke.log
timeout 600 python bench.py > gpurun_out/r75_b1.log 2>&1; echo "exit $?" >> gpurun_out/r75_b1.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 > gpurun_out/r75_b2.log 2>&1; echo "exit $?" >> gpurun_out/r75_b2.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 > gpurun_out/r75_b4.log 2>&1; echo "exit $?" >> gpurun_out/r75_b4.log
tail -n 2 gpurun_out/r75_tests.log gpurun_out/r75_smoke.log
