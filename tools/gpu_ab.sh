#!/bin/bash
# usage: bash tools/gpu_ab.sh "<cases>" "<pytest paths or ->" name1 name2 ...
# A/B of build variants (tools/gpu_variants.sh) preceded by the GPU tests on the in-tree library.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cases=$1; shift
tests=$1; shift
if [ "$tests" != "-" ]; then
  timeout 1200 python -m pytest $tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
rm -f gpurun_out/variants.log
bash tools/gpu_variants.sh "$cases" "$@"
