cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/attn_dbg.py > gpurun_out/r52_dbg.json 2>&1; echo "exit $?" >> gpurun_out/r52_dbg.json
cat gpurun_out/r52_dbg.json
