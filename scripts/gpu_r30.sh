cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export VARIANTS=1 VM=8192 VN=6400 VK=1600
for bn in 256 128; do MERAK_GEMM_BN=$bn timeout 120 python tools/gemm_bench.py > gpurun_out/r30_var_bn$bn.json 2>&1; done
for bn in 256 128; do
MERAK_GEMM_BN=$bn timeout 600 ncu --set full --clock-control none -k regex:gemm_kernel -s 3 -c 1 -o gpurun_out/r30_gemm_bn$bn -f python tools/gemm_bench.py > gpurun_out/r30_ncu_bn$bn.log 2>&1
done
cat gpurun_out/r30_var_*.json
