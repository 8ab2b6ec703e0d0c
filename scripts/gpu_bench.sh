cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/b_full.log 2>&1; echo "bench exit $?" >> gpurun_out/b_full.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/b_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ncu_launch.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_launch.log
timeout 900 python -m pytest tests/test_gpu_layer.py -q -m gpu --timeout 300 -p no:cacheprovider -k "ragged" > gpurun_out/r2_layer.log 2>&1
