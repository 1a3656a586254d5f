#!/bin/bash
# usage: bash tools/gpu_iter.sh "<perf cases>" [ncu_cfg ncu_prec]
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
TOR_DEBUG_TIMING=1 timeout 600 python tools/quick_perf.py "$1" > gpurun_out/quick_perf.log 2>&1
echo "perf exit $?" >> gpurun_out/quick_perf.log
if [ -n "$2" ]; then
  timeout 300 python tools/prof_one.py $2 $3 > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/prof_$4 python tools/prof_one.py $2 $3 > gpurun_out/ncu.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu.log
fi
