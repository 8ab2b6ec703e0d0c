cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export MERAK_AR_TIMEOUT_MS=10000
for rep in 1 2; do for P in 0 1; do
MERAK_CR_PRIO_HI=$P timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 297$rep$P bench.py --gpus 4 --no-cpu-baseline --no-extras > gpurun_out/r72_b4_${rep}_$P.log 2>&1
MERAK_CR_PRIO_HI=$P timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 298$rep$P bench.py --gpus 2 --no-cpu-baseline --no-extras > gpurun_out/r72_b2_${rep}_$P.log 2>&1
done; done
for f in gpurun_out/r72_*.log; do echo "$f $(grep '^{' $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_layer"],3))' 2>/dev/null)"; done
