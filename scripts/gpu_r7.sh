cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu --timeout 120 -p no:cacheprovider -x -k gemm > gpurun_out/r7_kern.log 2>&1; echo "exit $?" >> gpurun_out/r7_kern.log
timeout 120 python tools/gemm_bench.py > gpurun_out/r7_gemm_cg2.json 2>&1
MERAK_GEMM_CG=1 timeout 120 python tools/gemm_bench.py > gpurun_out/r7_gemm_cg1.json 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/r7_tests.log 2>&1; echo "exit $?" >> gpurun_out/r7_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r7_bench.log 2>&1
