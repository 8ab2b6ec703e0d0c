cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_chain.py -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/r57_tests.log 2>&1; echo "exit $?" >> gpurun_out/r57_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r57_b1.log 2>&1; echo "exit $?" >> gpurun_out/r57_b1.log
tail -n 2 gpurun_out/r57_tests.log
