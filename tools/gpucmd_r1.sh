cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 120 ./tools/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/quick_perf.py > gpurun_out/quick_perf.log 2>&1
echo "perf exit $?" >> gpurun_out/quick_perf.log
