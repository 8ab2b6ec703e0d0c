#!/bin/bash
# 1-GPU A/B of an environment switch on one box (alternating):  gpurun -- bash scripts/gpu_env_ab.sh VAR [bench args]
cd "${GRAFT_REPO_ROOT:-.}"
VAR=$1; shift
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for i in 1 2 3; do
  for v in 0 1; do
    env $VAR=$v timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 10 --warmup 3 "$@" > gpurun_out/eab_${v}_$i.json 2>> gpurun_out/eab.err
  done
done
