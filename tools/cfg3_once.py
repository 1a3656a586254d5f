"""One cfg3 batch (4096 x n=16) evaluation per precision, for launch lists (development aid)."""
import sys

sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402

ms = W.load_cfg3_batch(4096)
for prec in (sys.argv[1:] or ["fp64"]):
    T.torontonian_batch(ms[:64], prec)
    rs = T.torontonian_batch(ms, prec)
    print(prec, rs[0]["value"], rs[0].get("device_ms"), flush=True)
