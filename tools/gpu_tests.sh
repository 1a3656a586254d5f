#!/bin/bash
# GPU test pass: pytest -m gpu on the given test paths (default: all).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest ${@:-tests} -q -m gpu -x -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
