cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/gemm_bench.py > gpurun_out/r8_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/prof_gemm_cg2 -f python tools/gemm_bench.py > gpurun_out/r8_ncu.log 2>&1
echo "exit $?" >> gpurun_out/r8_ncu.log
