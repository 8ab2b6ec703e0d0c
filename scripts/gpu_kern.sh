#!/bin/bash
# kernel-level parity + microbenchmarks (GEMM at gpt20b shapes, attention):  gpurun -- bash scripts/gpu_kern.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -p no:cacheprovider > gpurun_out/kern_tests.log 2>&1
echo "exit $?" >> gpurun_out/kern_tests.log
H=6144 T=1 M_TOK=4096 CUBLAS=1 timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_bench.jsonl 2> gpurun_out/gemm_bench.err
H=6144 T=4 M_TOK=4096 CUBLAS=1 timeout 300 python tools/gemm_bench.py >> gpurun_out/gemm_bench.jsonl 2>> gpurun_out/gemm_bench.err
timeout 300 python tools/attn_time.py > gpurun_out/attn_time.json 2> gpurun_out/attn_time.err
