cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/r3_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r3_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r3_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/r3_bench.log
