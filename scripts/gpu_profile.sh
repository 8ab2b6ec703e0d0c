#!/bin/bash
# ncu evidence for profiles/ (one GPU; each ncu pass only after the plain command exited 0):
#   gpurun --timeout 3000 -- bash scripts/gpu_profile.sh [bench args]
# 1. the launch list of the bench step (gpu__time_duration per launch, serialised, cold cache);
# 2. --set full of the dominant kernels (GEMM, attention forward / backward, all-reduce epilogues).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras $*"
timeout 600 $CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
for k in gemm_kernel attn_fwd_tc_kernel attn_bwd_tc_kernel ar_fwd_kernel ar_bwd_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 2 \
    -o gpurun_out/prof_$k -f $CMD > gpurun_out/ncu_$k.log 2>&1
done
echo done > gpurun_out/prof_done
