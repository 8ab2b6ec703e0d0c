#!/bin/bash
# attention-backward experiment variants (extra -D flags), same box:  gpurun -- bash scripts/gpu_attn_var.sh "V1 V2 ..."
# each variant name maps to flags below; results in gpurun_out/attn_var.log
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1
SH=${SHAPES:-2,2048,64,96:4,1024,25,64}
: > gpurun_out/attn_var.log
for v in base ${1}; do
  case $v in
    base) F="";;
    nowait) F="-DABW_NO_WAIT";;
    nodq) F="-DABW_NO_DQ";;
    noexp) F="-DABW_NO_EXP";;
    noexp_nodq) F="-DABW_NO_EXP -DABW_NO_DQ";;
    *) F="$(echo $v | sed 's/,/ /g')";;
  esac
  if [ "$v" = base ]; then LIBV=$PWD/paper_2206_04959_b200/libmerak_tmp.so; else
    LIBV=$PWD/build/lib_$v.so
    MERAK_EXTRA_NVCC="$F" MERAK_LIB_OUT=$LIBV python -c 'import __graft_entry__ as g; g.build()' >> gpurun_out/build.log 2>&1
  fi
  for r in 1 2; do
    echo "$v $(MERAK_LIB=$LIBV timeout 120 python tools/attn_time.py $SH 2>&1 | python -c 'import sys,json
for l in sys.stdin:
  try: d=json.loads(l)
  except Exception: print(l.strip()); continue
  print(d["b"],d["s"],d["H"],d["d"],"fwd %.0f bwd %.0f us %.0f" % (d["fwd_tflops"], d["bwd_tflops"], d["bwd_us"]), end=" | ")')" >> gpurun_out/attn_var.log
  done
done
