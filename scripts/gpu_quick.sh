#!/bin/bash
# quick GPU check of selected test files:  gpurun -- bash scripts/gpu_quick.sh tests/test_x.py [...]
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest "$@" -x -q -m gpu -p no:cacheprovider -rs > gpurun_out/quick_tests.log 2>&1
echo "exit $?" >> gpurun_out/quick_tests.log
