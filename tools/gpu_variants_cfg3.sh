#!/bin/bash
# usage: bash tools/gpu_variants_cfg3.sh PREC name1 name2 ...   (name "default" = the in-tree library)
# Times one config-3 batch (tools/cfg3_once.py) per variants/lib_<name>.so, alternating 3 times.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
prec=$1; shift
for rep in 1 2 3; do
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=variants/lib_$v.so; fi
  echo "=== $v (rep $rep) $(TOR_B200_LIB=$lib timeout 300 python tools/cfg3_once.py $prec 2>&1 | tail -1)" >> gpurun_out/variants_cfg3.log
done
done
cat gpurun_out/variants_cfg3.log
