#!/bin/bash
# usage: bash tools/qd_variants.sh name1 name2 ...   (QD at n=28 of cfg4)
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  echo "=== $v" >> gpurun_out/variants.log
  TOR_B200_LIB=variants/lib_$v.so timeout 600 python tools/prof_one.py 4 256 28 >> gpurun_out/variants.log 2>&1
done
