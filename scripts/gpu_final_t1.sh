#!/bin/bash
# Round-end evidence on one B200: smoke, the default bench line, then the ncu launch list and --set full captures
# of the same bench command (scripts/gpu_profile.sh).   gpurun --timeout 3000 -- bash scripts/gpu_final_t1.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_final_t1.json 2> gpurun_out/bench_final_t1.err
echo "bench exit $?" >> gpurun_out/bench_final_t1.err
bash scripts/gpu_profile.sh
