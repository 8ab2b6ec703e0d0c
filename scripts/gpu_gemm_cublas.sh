#!/bin/bash
# GEMM vs cuBLAS at the gpt20b per-rank shapes (T = 1, 4, 8):  gpurun --timeout 900 -- bash scripts/gpu_gemm_cublas.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
: > gpurun_out/gemm_vs_cublas.jsonl
for T in 1 4 8; do
  CUBLAS=1 H=6144 T=$T M_TOK=4096 timeout 300 python tools/gemm_bench.py >> gpurun_out/gemm_vs_cublas.jsonl 2>> gpurun_out/gemm_vs_cublas.err
done
