"""One engine call for profiling: python tools/prof_one.py CFG PREC"""
import sys
sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402
cfg, prec = int(sys.argv[1]), sys.argv[2]
r = T.torontonian(W.load_config_instance(cfg), prec)
print(r["value"], r["kernel_ms"], r["device_ms"])
