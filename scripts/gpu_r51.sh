cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu --timeout 120 -p no:cacheprovider -k gemm -x > gpurun_out/r51_kern.log 2>&1; echo "exit $?" >> gpurun_out/r51_kern.log
tail -n 3 gpurun_out/r51_kern.log
grep -q "exit 0" gpurun_out/r51_kern.log || exit 1
timeout 600 python -m pytest tests/test_gpu_layer.py tests/test_gpu_chain.py -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/r51_layer.log 2>&1; echo "exit $?" >> gpurun_out/r51_layer.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r51_b1.log 2>&1; echo "exit $?" >> gpurun_out/r51_b1.log
MERAK_GEMM_DYN=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r51_b1_static.log 2>&1; echo "exit $?" >> gpurun_out/r51_b1_static.log
tail -n 2 gpurun_out/r51_layer.log
