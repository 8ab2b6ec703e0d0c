cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu --timeout 120 -p no:cacheprovider -x -k gemm > gpurun_out/r21_kern.log 2>&1; echo "exit $?" >> gpurun_out/r21_kern.log
timeout 120 python tools/gemm_bench.py > gpurun_out/r21_gemm.json 2>&1
for shp in "4096 4800 1600" "4096 1600 6400" "8192 6400 1600" "4096 1600 1600"; do
  set -- $shp
  VARIANTS=1 VM=$1 VN=$2 VK=$3 timeout 120 python tools/gemm_bench.py >> gpurun_out/r21_variants.json 2>&1
done
timeout 600 python -m pytest tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/r21_layer.log 2>&1; echo "exit $?" >> gpurun_out/r21_layer.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r21_bench.log 2>&1
