#!/bin/bash
# attention kernels: parity tests + microbenchmark (one GPU):  gpurun --timeout 900 -- bash scripts/gpu_attn.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -p no:cacheprovider -k attention > gpurun_out/attn_tests.log 2>&1
echo "exit $?" >> gpurun_out/attn_tests.log
timeout 300 python tools/attn_time.py > gpurun_out/attn_time.json 2> gpurun_out/attn_time.err
echo "exit $?" >> gpurun_out/attn_time.err
if [ "$1" == "full" ]; then
  timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/tests.log 2>&1
  echo "exit $?" >> gpurun_out/tests.log
fi
