cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/project_t8.py compute > gpurun_out/r77_t8_compute.json 2> gpurun_out/r77_t8_compute.err; echo "exit $?" >> gpurun_out/r77_t8_compute.err
tail -n 2 gpurun_out/r77_t8_compute.err
