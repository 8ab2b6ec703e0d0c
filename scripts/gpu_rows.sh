#!/bin/bash
# Row-kernel A/B (libmerak_base.so = previous build):  gpurun --timeout 900 -- bash scripts/gpu_rows.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
: > gpurun_out/row_bench.jsonl
for rep in 1 2; do
  MERAK_LIB=paper_2206_04959_b200/libmerak_base.so python tools/row_bench.py >> gpurun_out/row_bench.jsonl 2>> gpurun_out/row_bench.err
  python tools/row_bench.py >> gpurun_out/row_bench.jsonl 2>> gpurun_out/row_bench.err
done
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider > gpurun_out/rows_tests.log 2>&1
echo "exit $?" >> gpurun_out/rows_tests.log
