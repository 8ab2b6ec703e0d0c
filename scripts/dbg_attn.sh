cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
for sh in 4,1024,32,80 4,1024,8,80 1,256,2,80 4,1024,32,96 4,1024,25,64 2,2048,64,96 2,2048,8,128; do
  timeout 60 python tools/attn_time.py $sh >> gpurun_out/dbg_attn.json 2>> gpurun_out/dbg_attn.err
  echo "$sh exit $?" >> gpurun_out/dbg_attn.err
done
