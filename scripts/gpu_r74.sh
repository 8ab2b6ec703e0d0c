cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_ATTN_TC=1
for c in "1 128 1 64" "2 16 2 32" "2 100 3 64" "1 256 2 80" "2 1024 2 96" "1 192 2 128" "4 1024 4 64" "2 208 5 64" "2 2048 2 96"; do
  timeout 60 python tools/attn_bwd_case.py $c >> gpurun_out/r74_cases.log 2>&1 || echo "case $c FAILED rc=$?" >> gpurun_out/r74_cases.log
done
timeout 120 python tools/attn_bench.py > gpurun_out/r74_attn_tc.json 2>&1
MERAK_ATTN_TC=0 timeout 120 python tools/attn_bench.py > gpurun_out/r74_attn_mma.json 2>&1
grep case gpurun_out/r74_cases.log; cat gpurun_out/r74_attn_tc.json gpurun_out/r74_attn_mma.json
