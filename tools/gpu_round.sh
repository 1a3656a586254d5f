#!/bin/bash
# Round measurement pass: GPU tests, smoke, bench (engine + reference arm, driver form), other
# workloads, the launch list of the bench command and one ncu --set full capture of the DD kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for w in cfg4-n32-qd cfg3-batch-fp64 cfg3-batch-dd cfg5-n40-dd; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --cpu-sample-seconds 10 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
B="python bench.py --steps 1 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch exit $?" >> gpurun_out/ncu_launch.log
timeout 300 python tools/prof_one.py 4 128 > gpurun_out/prof_plain.log 2>&1 && \
timeout 1500 ncu --set full --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/prof_round python tools/prof_one.py 4 128 > gpurun_out/ncu_full.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_full.log
tail -2 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log
# QD (n = 28 sub-instance of config 4) and fp64 (config-3 batch) kernels: one ncu --set full capture each
bash tools/ncu_full.sh r02_qd_n28 4 256 28 > gpurun_out/ncu_qd.log 2>&1
bash tools/ncu_cfg3.sh r02_cfg3_fp64 fp64 > gpurun_out/ncu_cfg3.log 2>&1
for w in cfg1-n16-fp64 cfg2-n20-dd; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --cpu-sample-seconds 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
done
