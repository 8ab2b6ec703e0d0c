cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/r40_plain.log 2>&1; echo "plain exit $?" >> gpurun_out/r40_plain.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 528 -c 352 --csv --log-file gpurun_out/r40_launches.csv $CMD > gpurun_out/r40_ncu_launch.log 2>&1; echo "exit $?" >> gpurun_out/r40_ncu_launch.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 530 -c 4 -o gpurun_out/r40_gemm -f $CMD > gpurun_out/r40_ncu_gemm.log 2>&1; echo "exit $?" >> gpurun_out/r40_ncu_gemm.log
timeout 120 python tools/attn_bench.py > gpurun_out/r40_attn.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_bwd_dkdv_tc|attn_bwd_dq_tc|attn_fwd_kernel" -s 3 -c 3 -o gpurun_out/r40_attn -f python tools/attn_bench.py > gpurun_out/r40_ncu_attn.log 2>&1; echo "exit $?" >> gpurun_out/r40_ncu_attn.log
tail -n 1 gpurun_out/r40_ncu_launch.log gpurun_out/r40_ncu_gemm.log gpurun_out/r40_ncu_attn.log
