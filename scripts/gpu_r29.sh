cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for bn in 256 192 128; do MERAK_GEMM_BN=$bn timeout 120 python tools/gemm_bench.py > gpurun_out/r29_bn$bn.json 2>&1; done
MERAK_GEMM_BN=256 M_TOK=8192 timeout 120 python tools/gemm_bench.py > gpurun_out/r29_bn256_m8192.json 2>&1
MERAK_GEMM_BN=128 M_TOK=8192 timeout 120 python tools/gemm_bench.py > gpurun_out/r29_bn128_m8192.json 2>&1
