cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 900 python -m pytest tests/test_gpu_layer.py tests/test_gpu_multi.py -q -m gpu --timeout 800 -p no:cacheprovider > gpurun_out/r66_tests.log 2>&1; echo "exit $?" >> gpurun_out/r66_tests.log
tail -n 3 gpurun_out/r66_tests.log; grep -E "FAIL|not bit" gpurun_out/r66_tests.log | head
