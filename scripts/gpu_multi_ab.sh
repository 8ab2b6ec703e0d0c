#!/bin/bash
# multi-GPU A/B of an environment switch:  gpurun --gpus N -- bash scripts/gpu_multi_ab.sh N VAR
cd "${GRAFT_REPO_ROOT:-.}"
N=${1:-4}; VAR=${2:-MERAK_AR_FUSED_WAIT}
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
# the multi-process tests with the switch ON (its default is off)
env $VAR=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu -p no:cacheprovider -rs > gpurun_out/multi_tests_N${N}_$VAR.log 2>&1
echo "exit $?" >> gpurun_out/multi_tests_N${N}_$VAR.log
for i in 1 2; do
  for v in 0 1; do
    for CFG in gpt1.5b gpt20b; do
      env $VAR=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
        --master-port 29713 bench.py --gpus $N --config $CFG --steps 10 --warmup 3 --no-extras --no-cpu-baseline \
        > gpurun_out/mab_${CFG}_${v}_$i.json 2>> gpurun_out/mab.err
    done
  done
done
