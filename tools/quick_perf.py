"""Ad-hoc device timing of the engine through the public API (development aid)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402

cases = sys.argv[1].split(",") if len(sys.argv) > 1 else ["1:fp64", "1:128", "2:128", "2:256", "4:128"]
for c in cases:
    cfg, prec = c.split(":")
    m = W.load_config_instance(int(cfg))
    T.torontonian(m, prec)  # warm-up
    t0 = time.time()
    r = T.torontonian(m, prec)
    wall = time.time() - t0
    terms = r["term_count"]
    print(f"cfg{cfg} n={m.n_modes} {prec}: value={r['value']:.16e} words={r['words']} "
          f"kernel_ms={r['kernel_ms']:.3f} device_ms={r['device_ms']:.3f} wall={wall*1e3:.1f}ms "
          f"terms/s(device)={terms / (r['device_ms'] * 1e-3):.4e} canc={r['cancellation_bits']:.1f} "
          f"bits_left={r['bits_left']:.1f}", flush=True)
