#!/bin/bash
# GEMM raster A/B (auto band height vs the fixed 8-band): DRAM bytes per launch (ncu) and same-box bench values.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
[ -n "$SKIP_TESTS" ] || timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py -x -q -m gpu -p no:cacheprovider > gpurun_out/raster_tests.log 2>&1
echo "exit $?" >> gpurun_out/raster_tests.log
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras"
for G in ${GS:-4 8 16}; do
  MERAK_GEMM_GROUP_M=$G timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_g$G.csv $CMD > gpurun_out/ncu_g$G.log 2>&1
done
for i in 1 2 3; do
  for G in ${GS:-4 8 16}; do
    MERAK_GEMM_GROUP_M=$G timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/rab_${G}_$i.json 2>> gpurun_out/rab.err
  done
done
