#!/bin/bash
# usage: bash tools/gpu_variants.sh "<cases>" name1 name2 ...   (name "default" = the in-tree library)
# Runs tools/quick_perf.py (and, with CFG3=1, the cfg3 batch in fp64 and DD) on each
# variants/lib_<name>.so, alternating twice for A/B noise.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cases=$1; shift
for rep in 1 2; do
for v in "$@"; do
  echo "=== $v (rep $rep)" >> gpurun_out/variants.log
  if [ "$v" = default ]; then lib=""; else lib=variants/lib_$v.so; fi
  TOR_B200_LIB=$lib timeout 600 python tools/quick_perf.py "$cases" >> gpurun_out/variants.log 2>&1
  if [ -n "$CFG3" ]; then TOR_B200_LIB=$lib timeout 600 python tools/cfg3_once.py fp64 128 fp64 128 >> gpurun_out/variants.log 2>&1; fi
done
done
grep -E "===|kernel_ms|^fp64|^128" gpurun_out/variants.log | sed -E 's/value=[^ ]+ words=\([^)]*\) //'
