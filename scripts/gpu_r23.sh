cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_ATTN_TC=1
for c in "2 16 2 32" "2 100 3 64" "1 256 2 80" "2 1024 2 96" "1 192 2 128" "4 1024 4 64" "1 128 1 64" "1 64 1 64" "1 192 1 64"; do
  timeout 40 python tools/attn_case.py $c >> gpurun_out/r23_cases.log 2>&1 || echo "case $c FAILED/TIMEOUT rc=$?" >> gpurun_out/r23_cases.log
done
