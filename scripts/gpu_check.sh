#!/bin/bash
# Round-end style check on one B200 (run through gpurun from the repo root):
#   gpurun --timeout 3000 -- bash scripts/gpu_check.sh
# GPU parity tests (incl. the in-process T = 2/4/8 groups), smoke, bench, ncu launch list of the bench.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu -p no:cacheprovider -rs > gpurun_out/tests.log 2>&1
echo "tests exit $?" >> gpurun_out/tests.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
