cd "${GRAFT_REPO_ROOT:-.}"
for G in 4 8 16 64 148; do
  echo "G=$G $(MERAK_ATTN_BWD_GROUP=$G timeout 120 python tools/attn_time.py 2,2048,64,96:4,1024,25,64 2>&1 | python -c 'import sys,json
for l in sys.stdin:
  d=json.loads(l); print(d["b"],d["s"],d["H"],d["d"],"bwd %.0f us %.0f" % (d["bwd_tflops"], d["bwd_us"]), end=" | ")')" >> gpurun_out/attn_var.log
done
