#!/bin/bash
# All-reduce kernel CTA count sweep at T = N (gpt20b, push mode 2 default), interleaved:
#   gpurun --gpus N --timeout 1800 -- bash scripts/gpu_ctas_sweep.sh N
cd "${GRAFT_REPO_ROOT:-.}"
N=${1:-4}
mkdir -p gpurun_out
out=gpurun_out/ctas_sweep_N$N.txt
: > $out
for rep in 1 2; do
  for c in 0 32 74 148; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29732 \
      bench.py --gpus $N --config gpt20b --comm-ctas $c --steps 10 --warmup 3 --no-extras 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('comm_ctas=$c rep=$rep', round(d['value'],1), d['clocks']['sm_mhz'], round(d['ms_per_step'],3))" >> $out
  done
done
