cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_ATTN_TC=1
timeout 120 python tools/attn_bench.py > gpurun_out/r25_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_tc -s 3 -c 1 -o gpurun_out/prof_attn_tc2 -f python tools/attn_bench.py > gpurun_out/r25_ncu.log 2>&1
echo "exit $?" >> gpurun_out/r25_ncu.log
