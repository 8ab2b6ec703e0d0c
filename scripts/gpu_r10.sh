cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for shp in "4096 4800 1600" "4096 1600 6400" "8192 6400 1600" "4096 1600 1600"; do
  set -- $shp
  VARIANTS=1 VM=$1 VN=$2 VK=$3 timeout 120 python tools/gemm_bench.py >> gpurun_out/r10_variants.json 2>&1
done
