#!/bin/bash
# usage: bash tools/f64_variants.sh name1 name2 ...   (cfg1 + cfg3 batch in fp64 per variant)
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  echo "=== $v" >> gpurun_out/f64_variants.log
  TOR_B200_LIB=variants/lib_$v.so timeout 300 python tools/cfg3_once.py fp64 >> gpurun_out/f64_variants.log 2>&1
  TOR_B200_LIB=variants/lib_$v.so timeout 300 python tools/quick_perf.py "1:fp64" 2>&1 | grep -v "^\[tor\]" >> gpurun_out/f64_variants.log
done
