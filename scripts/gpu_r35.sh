cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 600 python -m pytest tests/test_gpu_fp32.py -q -m gpu --timeout 300 -p no:cacheprovider -s > gpurun_out/r35_fp32.log 2>&1; echo "exit $?" >> gpurun_out/r35_fp32.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 800 -p no:cacheprovider -s -k "2" > gpurun_out/r35_multi.log 2>&1; echo "exit $?" >> gpurun_out/r35_multi.log
tail -n 3 gpurun_out/r35_fp32.log gpurun_out/r35_multi.log
