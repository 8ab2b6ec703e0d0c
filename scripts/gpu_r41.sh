cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/attn_bench.py > gpurun_out/r41_attn.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_dkdv_tc -s 2 -c 1 -o gpurun_out/r41_dkdv -f python tools/attn_bench.py > gpurun_out/r41_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_dq_tc -s 2 -c 1 -o gpurun_out/r41_dq -f python tools/attn_bench.py > gpurun_out/r41_ncu2.log 2>&1
tail -n 1 gpurun_out/r41_ncu1.log gpurun_out/r41_ncu2.log
