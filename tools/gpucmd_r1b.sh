cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/prof_one.py 4 128 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:subtree -c 1 -o gpurun_out/prof_dd_n32 python tools/prof_one.py 4 128 > gpurun_out/ncu_dd.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_dd.log
