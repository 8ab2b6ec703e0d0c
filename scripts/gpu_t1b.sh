#!/bin/bash
# One B200: layer / kernel / group parity tests, then the N = 1 bench line.
#   gpurun --timeout 1500 -- bash scripts/gpu_t1b.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_group.py tests/test_gpu_chain.py \
  -x -q -m gpu -p no:cacheprovider > gpurun_out/t1b_tests.log 2>&1
echo "exit $?" >> gpurun_out/t1b_tests.log
timeout 600 python bench.py > gpurun_out/bench_t1b.json 2> gpurun_out/bench_t1b.err
echo "exit $?" >> gpurun_out/bench_t1b.err
