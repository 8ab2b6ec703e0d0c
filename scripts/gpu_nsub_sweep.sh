#!/bin/bash
# Sub-batch sweep n = 1 / 2 / 4 at T = N (BASELINE configs[4]: gpt20b, "sub-batch sweep 1/2/4"), interleaved:
#   gpurun --gpus N --timeout 1800 -- bash scripts/gpu_nsub_sweep.sh N
cd "${GRAFT_REPO_ROOT:-.}"
N=${1:-4}
mkdir -p gpurun_out
out=gpurun_out/nsub_sweep_N$N.txt
: > $out
for rep in 1 2; do
  for ns in 1 2 4; do
    if [ "$N" = "1" ]; then
      cmd="python bench.py"
    else
      cmd="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29730 bench.py --gpus $N"
    fi
    timeout 600 $cmd --config gpt20b --n-sub $ns --steps 10 --warmup 3 --no-extras --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('n_sub=$ns rep=$rep', round(d['value'],1), d['clocks']['sm_mhz'], round(d['ms_per_step'],3))" >> $out
  done
done
