"""One engine call for profiling: python tools/prof_one.py CFG PREC [MODES]
MODES: use the first MODES click modes of the config instance (sub-Torontonian)."""
import sys
sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import matrix as M  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402
cfg, prec = int(sys.argv[1]), sys.argv[2]
m = W.load_config_instance(cfg)
if len(sys.argv) > 3:
    m = M.select_modes(m, list(range(int(sys.argv[3]))))
r = T.torontonian(m, prec)
print(r["value"], r["kernel_ms"], r["device_ms"])
