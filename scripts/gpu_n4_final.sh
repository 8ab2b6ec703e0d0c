#!/bin/bash
# Full GPU test suite on a 4-GPU box (multi-process tests included), the N = T = 4 gpt20b bench line and the
# NVLink byte counters:   gpurun --gpus 4 --timeout 2400 -- bash scripts/gpu_n4_final.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider -rs > gpurun_out/tests_4gpu.log 2>&1
echo "tests exit $?" >> gpurun_out/tests_4gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29720 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_final_N4.json 2> gpurun_out/bench_final_N4.err
echo "exit $?" >> gpurun_out/bench_final_N4.err
for mode in 0 2; do
  env MERAK_AR_PUSH=$mode timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 29722 tools/nvlink_bytes.py > gpurun_out/nvlink_bytes_push${mode}_N4.json \
    2> gpurun_out/nvlink_bytes_push${mode}_N4.err
done
