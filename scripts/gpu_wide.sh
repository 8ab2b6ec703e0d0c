#!/bin/bash
# Backward-epilogue variant check on one B200:  gpurun --timeout 1500 -- bash scripts/gpu_wide.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
python tools/row_bench.py > gpurun_out/row_bench_wide.jsonl 2> gpurun_out/row_bench_wide.err
python tools/row_bench.py >> gpurun_out/row_bench_wide.jsonl 2>> gpurun_out/row_bench_wide.err
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_push.py tests/test_gpu_chain.py \
  tests/test_gpu_recompute.py -x -q -m gpu -p no:cacheprovider > gpurun_out/wide_tests.log 2>&1
echo "exit $?" >> gpurun_out/wide_tests.log
timeout 600 python bench.py > gpurun_out/bench_wide.json 2> gpurun_out/bench_wide.err
