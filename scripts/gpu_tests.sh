cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r1_smi.log 2>&1
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -m gpu --timeout 120 -p no:cacheprovider > gpurun_out/r1_kern.log 2>&1
echo "kern exit $?" >> gpurun_out/r1_kern.log
timeout 900 python -m pytest tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider -s > gpurun_out/r1_layer.log 2>&1
echo "layer exit $?" >> gpurun_out/r1_layer.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r1_smoke.log
