#!/bin/bash
# ncu --set full of the fp64 / DD subtree kernel on the config-3 batch: bash tools/ncu_cfg3.sh NAME PREC
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/cfg3_once.py $2 > gpurun_out/$1_plain.log 2>&1 || { cat gpurun_out/$1_plain.log; exit 1; }
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:subtree -s 1 -c 1 \
  --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum \
  -o gpurun_out/$1 python tools/cfg3_once.py $2 > gpurun_out/$1_ncu.log 2>&1
echo "ncu exit $?"; cat gpurun_out/$1_plain.log
