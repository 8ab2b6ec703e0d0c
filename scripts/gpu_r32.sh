cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/r32_layer.log 2>&1; echo "layer exit $?" >> gpurun_out/r32_layer.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r32_b1.log 2>&1; echo "bench exit $?" >> gpurun_out/r32_b1.log
MERAK_STREAMS=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r32_b1_single.log 2>&1; echo "bench exit $?" >> gpurun_out/r32_b1_single.log
tail -n 2 gpurun_out/r32_layer.log
