cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export T8_CONFIGS=gpt20b
( timeout 240 python tools/project_t8.py compute > gpurun_out/r47_a.json 2> gpurun_out/r47_a.err; echo "exit $?" >> gpurun_out/r47_a.err ) &
P=$!
for i in 1 2 3 4 5 6 7 8; do sleep 25; nvidia-smi --query-gpu=utilization.gpu,power.draw,clocks.sm --format=csv,noheader >> gpurun_out/r47_smi.log; done
wait $P
MERAK_STREAMS=1 timeout 240 python tools/project_t8.py compute > gpurun_out/r47_b.json 2> gpurun_out/r47_b.err; echo "exit $?" >> gpurun_out/r47_b.err
tail -n 3 gpurun_out/r47_a.err gpurun_out/r47_b.err gpurun_out/r47_smi.log
