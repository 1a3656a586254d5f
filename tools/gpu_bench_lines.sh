#!/bin/bash
# The committed bench lines of a round: the driver's command, the reference arm and every other workload.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
for w in cfg4-n32-qd cfg3-batch-fp64 cfg3-batch-dd cfg5-n40-dd cfg1-n16-fp64 cfg2-n20-dd; do
  st=3; [ "$w" = cfg1-n16-fp64 -o "$w" = cfg2-n20-dd ] && st=20
  [ "${w:0:10}" = cfg3-batch ] && st=10
  timeout 900 python bench.py --workload $w --steps $st --warmup 3 --cpu-sample-seconds 10 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w exit $?"
done
