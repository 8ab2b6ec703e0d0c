cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in "1 128 1 64" "2 16 2 32" "2 100 3 64" "1 256 2 80" "2 1024 2 96" "1 192 2 128" "4 1024 4 64" "2 208 5 64"; do
  timeout 60 python tools/attn_bwd_case.py $c >> gpurun_out/r42_cases.log 2>&1 || echo "case $c FAILED rc=$?" >> gpurun_out/r42_cases.log
done
timeout 120 python tools/attn_bench.py > gpurun_out/r42_attn.json 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/r42_tests.log 2>&1; echo "exit $?" >> gpurun_out/r42_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r42_b1.log 2>&1; echo "exit $?" >> gpurun_out/r42_b1.log
grep case gpurun_out/r42_cases.log; cat gpurun_out/r42_attn.json; tail -n 2 gpurun_out/r42_tests.log
