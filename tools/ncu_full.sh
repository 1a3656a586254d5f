#!/bin/bash
# One ncu --set full capture of the subtree kernel: bash tools/ncu_full.sh NAME CFG PREC [MODES]
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
name=$1; shift
timeout 300 python tools/prof_one.py "$@" > gpurun_out/${name}_plain.log 2>&1 || { echo "plain run failed"; cat gpurun_out/${name}_plain.log; exit 1; }
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:subtree -c 1 \
  --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -o gpurun_out/${name} python tools/prof_one.py "$@" > gpurun_out/${name}_ncu.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/${name}_ncu.log; cat gpurun_out/${name}_plain.log
