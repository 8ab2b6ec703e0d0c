cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu --timeout 120 -p no:cacheprovider -k attention > gpurun_out/r11_kern.log 2>&1; echo "exit $?" >> gpurun_out/r11_kern.log
timeout 120 python tools/attn_bench.py > gpurun_out/r11_attn_tc.json 2>&1
MERAK_ATTN_TC=0 timeout 120 python tools/attn_bench.py > gpurun_out/r11_attn_old.json 2>&1
