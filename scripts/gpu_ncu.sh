cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/ncu_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 20 -c 6 -o gpurun_out/prof_gemm -f $CMD > gpurun_out/ncu_gemm.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn|ar_|colsum|sample_reduce" -s 30 -c 8 -o gpurun_out/prof_misc -f $CMD > gpurun_out/ncu_misc.log 2>&1
echo "exit $?" >> gpurun_out/ncu_misc.log
