#!/bin/bash
# usage: bash tools/gpu_qd_ab.sh name1 name2 ...: QD n=28 sub-instance of config 4 per library variant (twice)
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=variants/lib_$v.so; fi
  echo -n "$v: "; TOR_B200_LIB=$lib timeout 600 python tools/prof_one.py 4 256 28
done; done
