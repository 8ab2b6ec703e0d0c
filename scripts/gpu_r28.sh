cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu --timeout 120 -p no:cacheprovider > gpurun_out/r28_kern.log 2>&1; echo "kern exit $?" >> gpurun_out/r28_kern.log
timeout 900 python -m pytest tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/r28_layer.log 2>&1; echo "layer exit $?" >> gpurun_out/r28_layer.log
timeout 600 python bench.py > gpurun_out/r28_b1.log 2>&1; echo "bench exit $?" >> gpurun_out/r28_b1.log
tail -3 gpurun_out/r28_kern.log gpurun_out/r28_layer.log; tail -2 gpurun_out/r28_b1.log
