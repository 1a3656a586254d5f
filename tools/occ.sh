cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
TOR_DEBUG_TIMING=1 timeout 300 python tools/quick_perf.py 4:128 2>&1 | grep -E "cfg|subtree_kernel|smem 0 " >> gpurun_out/occ.log
for b in 2; do echo "== bps $b" >> gpurun_out/occ.log; TOR_BLOCKS_PER_SM=$b timeout 300 python tools/quick_perf.py 4:128 2>&1 | grep -E "cfg" >> gpurun_out/occ.log; done
