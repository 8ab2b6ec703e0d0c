cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 900 python tools/project_t8.py compute > gpurun_out/r46_t8_compute.json 2> gpurun_out/r46_t8_compute.err; echo "exit $?" >> gpurun_out/r46_t8_compute.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tools/project_t8.py comm > gpurun_out/r46_t8_comm.json 2> gpurun_out/r46_t8_comm.err; echo "exit $?" >> gpurun_out/r46_t8_comm.err
tail -n 1 gpurun_out/r46_t8_compute.err gpurun_out/r46_t8_comm.err
