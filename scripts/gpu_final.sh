cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/f_tests.log 2>&1; echo "exit $?" >> gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1; echo "exit $?" >> gpurun_out/f_smoke.log
timeout 600 python bench.py > gpurun_out/f_b1.log 2>&1; echo "exit $?" >> gpurun_out/f_b1.log
timeout 600 python bench.py --impl reference > gpurun_out/f_ref.log 2>&1; echo "exit $?" >> gpurun_out/f_ref.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 > gpurun_out/f_b2.log 2>&1; echo "exit $?" >> gpurun_out/f_b2.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 > gpurun_out/f_b4.log 2>&1; echo "exit $?" >> gpurun_out/f_b4.log
for n in 1 2; do NSUB=$n timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2954$n tools/timeline.py > gpurun_out/f_tl2_n$n.log 2>&1; done
LPS=$(grep '^{' gpurun_out/f_b1.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['gpu_launches']//d['steps'])")
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extras"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s $((3*LPS)) -c $((2*LPS+2)) --csv --log-file gpurun_out/f_launches.csv $CMD > gpurun_out/f_ncu.log 2>&1; echo "exit $? LPS=$LPS" >> gpurun_out/f_ncu.log
tail -n 2 gpurun_out/f_tests.log gpurun_out/f_smoke.log gpurun_out/f_ncu.log
