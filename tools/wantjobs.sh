#!/bin/bash
cd $GRAFT_REPO_ROOT
for w in ${WJ:-65536 131072 262144 524288}; do
  echo "=== want $w" >> gpurun_out/variants.log
  TOR_WANT_JOBS=$w timeout 600 python tools/quick_perf.py 4:128 >> gpurun_out/variants.log 2>&1
done
