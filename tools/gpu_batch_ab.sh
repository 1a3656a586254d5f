#!/bin/bash
# usage: bash tools/gpu_batch_ab.sh name1 name2 ...: cfg3 batch bench lines (fp64, DD) per library variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = default ]; then lib=""; else lib=variants/lib_$v.so; fi
  for w in cfg3-batch-fp64 cfg3-batch-dd; do
    TOR_B200_LIB=$lib timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2> gpurun_out/bab.err | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$v $w device_ms', round(d['ms_per_step'],3), 'e2e_ms', round(d['e2e']['ms_per_step'],3), 'ratio', round(d['e2e']['over_device'],2), 'item0', d['result']['item0'])"
  done
done
