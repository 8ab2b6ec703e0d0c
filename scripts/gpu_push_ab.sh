#!/bin/bash
# Interleaved A/B of the all-reduce variants at T = N (gpt20b, no extras), then NVLink byte counters:
#   gpurun --gpus N --timeout 1800 -- bash scripts/gpu_push_ab.sh N
cd "${GRAFT_REPO_ROOT:-.}"
N=${1:-4}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
out=gpurun_out/push_ab_N$N.txt
: > $out
for rep in 1 2 3; do
  for mode in 0 1 2; do
    env MERAK_AR_PUSH=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29716 bench.py --gpus $N --config gpt20b --steps 10 --warmup 3 \
      --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('push=$mode rep=$rep', round(d['value'],1), d['clocks']['sm_mhz'], d['ms_per_step'])" >> $out
  done
done
for mode in 0 2; do
  env MERAK_AR_PUSH=$mode timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29718 tools/nvlink_bytes.py > gpurun_out/nvlink_bytes_push${mode}_N$N.json \
    2> gpurun_out/nvlink_bytes_push${mode}_N$N.err
done
