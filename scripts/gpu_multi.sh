#!/bin/bash
# Multi-GPU check on N GPUs of one box:  gpurun --gpus N --timeout 2400 -- bash scripts/gpu_multi.sh N
# multi-process parity (peer all-reduce + NCCL baseline) and the bench line at T = N (gpt20b headline,
# gpt1.5b side workload), plus the all-reduce microbenchmark inside bench.py.
cd "${GRAFT_REPO_ROOT:-.}"
N=${1:-2}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -p no:cacheprovider -rs > gpurun_out/multi_tests_N$N.log 2>&1
echo "exit $?" >> gpurun_out/multi_tests_N$N.log
for CFG in ${CFGS:-gpt20b gpt1.5b}; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29712 \
    bench.py --gpus $N --config $CFG --steps 10 --warmup 3 > gpurun_out/bench_${CFG}_N$N.json 2> gpurun_out/bench_${CFG}_N$N.err
  echo "exit $?" >> gpurun_out/bench_${CFG}_N$N.err
done
