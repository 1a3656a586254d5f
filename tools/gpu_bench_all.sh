#!/bin/bash
# Bench lines of every workload (engine arm) into gpurun_out/bench_<workload>.json
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in ${@:-cfg4-n32-dd cfg3-batch-fp64 cfg3-batch-dd cfg1-n16-fp64 cfg2-n20-dd cfg4-n32-qd}; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --cpu-sample-seconds 10 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "$w exit $?"; tail -c 400 gpurun_out/bench_$w.json
done
