cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in "2 100 3 64" "4 1024 4 64" "2 208 5 64" "2 16 2 32"; do
  timeout 60 python tools/attn_bwd_case.py $c >> gpurun_out/r43_cases.log 2>&1 || echo "case $c FAILED rc=$?" >> gpurun_out/r43_cases.log
done
timeout 120 python tools/attn_bench.py > gpurun_out/r43_attn.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_bwd -c 8 --csv python tools/attn_bench.py > gpurun_out/r43_ncu.csv 2>&1
grep case gpurun_out/r43_cases.log; cat gpurun_out/r43_attn.json; grep -E "attn_bwd" gpurun_out/r43_ncu.csv | awk -F'","' '{print $5, $NF}' | cut -c1-120
