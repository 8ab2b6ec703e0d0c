#!/bin/bash
# Fused GEMM -> reduce-scatter push on N GPUs:  gpurun --gpus N --timeout 1800 -- bash scripts/gpu_push.sh N
# multi-process parity (incl. the push over NVLink), then the gpt20b bench line at T = N with the push pass, and
# an A/B of the main line with MERAK_AR_PUSH=1.
cd "${GRAFT_REPO_ROOT:-.}"
N=${1:-2}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_push.py -x -q -m gpu -p no:cacheprovider -rs > gpurun_out/push_tests_N$N.log 2>&1
echo "exit $?" >> gpurun_out/push_tests_N$N.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29714 bench.py --gpus $N --config gpt20b --steps 10 --warmup 3 ${BENCH_ARGS} \
    > gpurun_out/bench_${name}_N$N.json 2> gpurun_out/bench_${name}_N$N.err
  echo "exit $?" >> gpurun_out/bench_${name}_N$N.err
}
run main MERAK_BENCH_NONE=1
BENCH_ARGS=--no-extras run push_main MERAK_AR_PUSH=1 MERAK_AR_TWO_SHOT=1
BENCH_ARGS=--no-extras run pushag_main MERAK_AR_PUSH=2 MERAK_AR_TWO_SHOT=1
BENCH_ARGS=--no-extras run pull_main2 MERAK_BENCH_NONE=1
