cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --timeout 800 -p no:cacheprovider -s > gpurun_out/r73_multi.log 2>&1; echo "exit $?" >> gpurun_out/r73_multi.log
tail -n 2 gpurun_out/r73_multi.log; grep -E "d80 T=|d96 T=" gpurun_out/r73_multi.log | head -4 | cut -c1-200
