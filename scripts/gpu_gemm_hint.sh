#!/bin/bash
# GEMM L2 eviction-hint sweep (MERAK_GEMM_HINT="abc"): DRAM bytes per launch (ncu) and same-box bench values.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
HS=${HS:-000 001 201 021}
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras"
for H in $HS; do
  MERAK_GEMM_HINT=$H timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_h$H.csv $CMD > gpurun_out/ncu_h$H.log 2>&1
done
for i in $(seq 1 ${R:-2}); do
  for H in $HS; do
    MERAK_GEMM_HINT=$H timeout 600 python bench.py --no-extras --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/hab_${H}_$i.json 2>> gpurun_out/hab.err
  done
done
