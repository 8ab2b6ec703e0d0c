cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras"
timeout 300 $CMD > gpurun_out/r76_plain.log 2>&1
LPS=$(grep '^{' gpurun_out/r76_plain.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['gpu_launches']//d['steps'])")
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $((3*LPS)) -c $((2*LPS+2)) --csv --log-file gpurun_out/r76_launches.csv $CMD > gpurun_out/r76_ncu.log 2>&1; echo "exit $? LPS=$LPS" >> gpurun_out/r76_ncu.log
tail -n 1 gpurun_out/r76_ncu.log
