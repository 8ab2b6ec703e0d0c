#!/bin/bash
# Interleaved A/B of environment switches at T = N (gpt20b, no extras):
#   gpurun --gpus N --timeout 1800 -- bash scripts/gpu_env_ab4.sh N "VAR=V[,VAR=V]" ...
cd "${GRAFT_REPO_ROOT:-.}"
N=$1; shift
mkdir -p gpurun_out
out=gpurun_out/env_ab_N$N.txt
: > $out
for rep in 1 2 3; do
  for v in "default" "$@"; do
    envs=""
    [ "$v" != "default" ] && envs=$(echo "$v" | tr ',' ' ')
    env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port 29728 bench.py --gpus $N --config gpt20b --steps 10 --warmup 3 --no-extras 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v rep=$rep', round(d['value'],1), d['clocks']['sm_mhz'], round(d['ms_per_step'],3))" >> $out
  done
done
