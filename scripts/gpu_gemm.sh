#!/bin/bash
# GEMM microbenchmarks at the layer shapes: gpurun -- bash scripts/gpu_gemm.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for T in 1 4 8; do
  for BN in 256 192 128; do
    H=6144 T=$T M_TOK=4096 MERAK_GEMM_BN=$BN CUBLAS=1 timeout 300 python tools/gemm_bench.py >> gpurun_out/gemm_bench.jsonl 2>> gpurun_out/gemm_bench.err
  done
done
