cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
fails=0
for i in $(seq 1 10); do
timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700+i)) bench.py --gpus 4 --no-cpu-baseline --no-extras --steps 40 > gpurun_out/r71_b4_$i.log 2>&1; rc=$?
echo "b4 $i rc=$rc $(grep '^{' gpurun_out/r71_b4_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))' 2>/dev/null)"
[ $rc -ne 0 ] && fails=$((fails+1))
done
for i in $(seq 1 12); do
timeout 150 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29800+i)) bench.py --gpus 2 --no-cpu-baseline --no-extras --steps 40 > gpurun_out/r71_b2_$i.log 2>&1; rc=$?
echo "b2 $i rc=$rc $(grep '^{' gpurun_out/r71_b2_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1))' 2>/dev/null)"
[ $rc -ne 0 ] && fails=$((fails+1))
done
echo "fails=$fails"
