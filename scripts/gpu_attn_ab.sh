#!/bin/bash
# Attention A/B (libmerak_base.so = the alternative build):  gpurun --timeout 900 -- bash scripts/gpu_attn_ab.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
: > gpurun_out/attn_ab.jsonl
for rep in 1 2; do
  MERAK_LIB=paper_2206_04959_b200/libmerak_base.so python tools/attn_time.py | sed 's/^/base /' >> gpurun_out/attn_ab.jsonl 2>> gpurun_out/attn_ab.err
  python tools/attn_time.py | sed 's/^/new /' >> gpurun_out/attn_ab.jsonl 2>> gpurun_out/attn_ab.err
done
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_recompute.py -x -q -m gpu -p no:cacheprovider > gpurun_out/attn_ab_tests.log 2>&1
echo "exit $?" >> gpurun_out/attn_ab_tests.log
