cd $GRAFT_REPO_ROOT
timeout 300 python tools/prof_one.py 4 128 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/prof_$1 python tools/prof_one.py 4 128 > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full.log
