cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -p no:cacheprovider -k attention > gpurun_out/attn_tests.log 2>&1
echo "exit $?" >> gpurun_out/attn_tests.log
timeout 120 python tools/attn_time.py > gpurun_out/attn_time.json 2>> gpurun_out/attn_time.err
for X in 0; do
  MERAK_ATTN_BWD_EXP=$X timeout 120 python tools/attn_dbg.py 2,2048,64,96 >> gpurun_out/attn_dbg.json 2>> gpurun_out/attn_dbg.err
done
