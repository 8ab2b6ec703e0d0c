cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 600 python -m pytest tests/test_gpu_chain.py -q -m gpu --timeout 300 -p no:cacheprovider -s > gpurun_out/r44_chain.log 2>&1; echo "exit $?" >> gpurun_out/r44_chain.log
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 800 -p no:cacheprovider -s -k "2" > gpurun_out/r44_multi.log 2>&1; echo "exit $?" >> gpurun_out/r44_multi.log
grep -E "^\{|passed|failed|exit" gpurun_out/r44_chain.log | cut -c1-600; grep -E "chain|FAIL|passed|failed" gpurun_out/r44_multi.log | head
