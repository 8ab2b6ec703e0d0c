cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_ATTN_TC=1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu --timeout 120 -p no:cacheprovider -k attention > gpurun_out/r22_kern.log 2>&1; echo "exit $?" >> gpurun_out/r22_kern.log
timeout 120 python tools/attn_bench.py > gpurun_out/r22_attn_tc.json 2>&1
