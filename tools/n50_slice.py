"""The paper's n = 50 (100 x 100) case as checkpointable prefix-class slices: one DD slice of
2^(50-k) subsets on one GPU, its device time and throughput (config 5's m = 100 state with
its 40 click modes plus the 10 lowest unused ones).  usage: python tools/n50_slice.py [k] [cls]"""
import sys
import time

sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402
from paper_2009_01177_b200.matrix import select_modes  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 12
cls = int(sys.argv[2]) if len(sys.argv) > 2 else 0x5a5
sel = set(W.click_set(5))
extra = [j for j in range(100) if j not in sel][:10]
m = select_modes(W.full_state(5), sorted(sel | set(extra)))
pl = T.api.Plan(m, "128", k, cls, cls + 1)
pl.execute()
t0 = time.time()
r = pl.execute()
wall = time.time() - t0
pl.close()
terms = 1 << (50 - k)
print(f"n=50 DD slice k={k} class {cls:#x}: {terms} subsets, device {r['device_ms']:.1f} ms "
      f"(kernel {r['kernel_ms']:.1f}), {terms / (r['device_ms'] * 1e-3):.4e} terms/s, wall {wall:.2f} s; "
      f"words {r['words']} sum|t| {r['sum_abs_terms']:.4e}; whole n=50 on one GPU at this rate: "
      f"{2 ** 50 / (terms / (r['device_ms'] * 1e-3)) / 3600:.2f} h, on 8: "
      f"{2 ** 50 / (terms / (r['device_ms'] * 1e-3)) / 3600 / 8:.2f} h", flush=True)
