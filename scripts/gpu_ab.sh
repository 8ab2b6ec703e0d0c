#!/bin/bash
# A/B of two in-tree builds on one box (alternating):  gpurun -- bash scripts/gpu_ab.sh [bench args]
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in prev new; do
    if [ $v == prev ]; then L=paper_2206_04959_b200/libmerak_tmp_prev.so; else L=paper_2206_04959_b200/libmerak_tmp.so; fi
    MERAK_LIB=$PWD/$L timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 20 --warmup 5 "$@" > gpurun_out/ab_${v}_$i.json 2>> gpurun_out/ab.err
  done
done
