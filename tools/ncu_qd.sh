#!/bin/bash
# QD profile at n=28 (sub-instance of cfg4)
cd $GRAFT_REPO_ROOT
TOR_DEBUG_TIMING=1 timeout 300 python tools/prof_one.py 4 256 28 > gpurun_out/prof_qd_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/prof_qd python tools/prof_one.py 4 256 28 > gpurun_out/ncu_qd.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_qd.log
