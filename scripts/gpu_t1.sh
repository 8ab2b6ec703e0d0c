#!/bin/bash
# One B200: the N = 1 bench line (gpt20b headline + T = 8 shard class breakdown), then T = 8 shard variants.
#   gpurun --timeout 1500 -- bash scripts/gpu_t1.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_t1.json 2> gpurun_out/bench_t1.err
echo "exit $?" >> gpurun_out/bench_t1.err
timeout 600 python tools/shard_time.py "" MERAK_GEMM_SMEM_KB=192 MERAK_GEMM_PICK_BN=1 MERAK_GEMM_DYN=1 \
  > gpurun_out/shard_time.jsonl 2> gpurun_out/shard_time.err
