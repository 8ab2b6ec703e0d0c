cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/r34_b1.log 2>&1; echo "exit $?" >> gpurun_out/r34_b1.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r34_ref.log 2>&1; echo "exit $?" >> gpurun_out/r34_ref.log
