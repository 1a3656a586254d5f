#!/bin/bash
# usage: bash tools/gpu_variants.sh "<cases>" name1 name2 ...
cd $GRAFT_REPO_ROOT
cases=$1; shift
for v in "$@"; do
  echo "=== $v" >> gpurun_out/variants.log
  TOR_B200_LIB=variants/lib_$v.so timeout 600 python tools/quick_perf.py "$cases" >> gpurun_out/variants.log 2>&1
done
