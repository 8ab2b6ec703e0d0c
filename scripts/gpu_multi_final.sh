#!/bin/bash
# N-GPU round-end evidence: multi-process parity tests, the gpt20b bench line at T = N, and an interleaved
# pull / push A/B.   gpurun --gpus N --timeout 2400 -- bash scripts/gpu_multi_final.sh N
cd "${GRAFT_REPO_ROOT:-.}"
N=${1:-4}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_push.py -x -q -m gpu -p no:cacheprovider -rs > gpurun_out/multi_final_N$N.log 2>&1
echo "exit $?" >> gpurun_out/multi_final_N$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29724 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/bench_multi_final_N$N.json 2> gpurun_out/bench_multi_final_N$N.err
echo "exit $?" >> gpurun_out/bench_multi_final_N$N.err
out=gpurun_out/push_ab_final_N$N.txt
: > $out
for rep in 1 2; do
  for mode in 0 2; do
    env MERAK_AR_PUSH=$mode MERAK_AR_TWO_SHOT=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29726 bench.py --gpus $N --config gpt20b --steps 10 --warmup 3 \
      --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('push=$mode two_shot=1 rep=$rep', round(d['value'],1), d['clocks']['sm_mhz'], d['ms_per_step'])" >> $out
  done
done
