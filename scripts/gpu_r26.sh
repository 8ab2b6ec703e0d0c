#!/bin/bash
# tcgen05 attention backward: correctness per case (each under its own timeout), then microbench
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
export MERAK_ATTN_BWD_TC=1
for c in "1 128 1 64" "2 16 2 32" "2 100 3 64" "1 256 2 80" "2 1024 2 96" "1 192 2 128" "4 1024 4 64" "2 208 5 64"; do
  timeout 60 python tools/attn_bwd_case.py $c >> gpurun_out/r26_cases.log 2>&1 || echo "case $c FAILED rc=$?" >> gpurun_out/r26_cases.log
done
MERAK_ATTN_BWD_TC=0 timeout 120 python tools/attn_bench.py > gpurun_out/r26_attn_old.json 2>&1
timeout 120 python tools/attn_bench.py > gpurun_out/r26_attn_bwdtc.json 2>&1
cat gpurun_out/r26_cases.log gpurun_out/r26_attn_*.json
