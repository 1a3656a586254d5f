"""Where the end-to-end time of one tor_torontonian call goes (development aid)."""
import os
import sys
import time
sys.path.insert(0, ".")
os.environ["TOR_DEBUG_TIMING"] = "1"
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402
m = W.load_config_instance(4)
for i in range(4):
    t0 = time.perf_counter()
    r = T.torontonian(m, "128")
    t1 = time.perf_counter()
    print(f"call {i}: wall {1e3*(t1-t0):.2f} ms  device_ms {r['device_ms']:.2f} kernel_ms {r['kernel_ms']:.2f}", flush=True)
t0 = time.perf_counter()
cfg = T.select_precision(m)
print(f"select_precision {1e3*(time.perf_counter()-t0):.2f} ms")
