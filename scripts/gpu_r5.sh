cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/r5_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/r5_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r5_bench.log 2>&1; echo "bench exit $?" >> gpurun_out/r5_bench.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches5.csv $CMD > gpurun_out/ncu_launch.log 2>&1
