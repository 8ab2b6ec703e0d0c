cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "exit $?" >> gpurun_out/r2c_bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2c_ref.json 2> gpurun_out/r2c_ref.err
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -p no:cacheprovider -k attention > gpurun_out/r2c_attn.log 2>&1
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_case.py single > gpurun_out/r2c_san_${t}_single.log 2>&1; echo "exit $?" >> gpurun_out/r2c_san_${t}_single.log
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py group > gpurun_out/r2c_san_memcheck_group.log 2>&1; echo "exit $?" >> gpurun_out/r2c_san_memcheck_group.log
