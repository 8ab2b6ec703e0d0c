cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider -x > gpurun_out/r9_tests.log 2>&1; echo "exit $?" >> gpurun_out/r9_tests.log
timeout 120 python tools/gemm_bench.py > gpurun_out/r9_gemm.json 2>&1
timeout 600 python bench.py > gpurun_out/r9_bench.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/r9_plain.log 2>&1 && \
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_kernel -s 72 -c 24 --csv --log-file gpurun_out/r9_gemm_dram.csv $CMD > gpurun_out/r9_ncu.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r9_launches.csv $CMD > gpurun_out/r9_ncu2.log 2>&1
echo "exit $?" >> gpurun_out/r9_ncu2.log
