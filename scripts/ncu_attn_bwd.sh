#!/bin/bash
# ncu --set full of the attention backward kernel at the gpt20b sub-batch shape (one launch):
#   gpurun -- bash scripts/ncu_attn_bwd.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
timeout 120 python tools/attn_time.py 2,2048,64,96 > gpurun_out/attn_time_pre_ncu.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_tc_kernel -s 3 -c 1 \
  -o gpurun_out/attn_bwd_full -f python tools/attn_time.py 2,2048,64,96 > gpurun_out/ncu_attn_bwd.log 2>&1
echo "exit $?" >> gpurun_out/ncu_attn_bwd.log
