"""Per-shard device time of the n=32 DD plan at 1/2/4/8-way prefix-class sharding on ONE
GPU (each shard run alone, as one rank of a P-GPU job would), and the fold of the shard
partials vs the unsharded result (development aid for the scaling figures)."""
import sys

sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prec = sys.argv[2] if len(sys.argv) > 2 else "128"
m = W.load_config_instance(cfg)
whole = None
for k in (0, 1, 2, 3):
    P = 1 << k
    worst, parts = 0.0, []
    for r in range(P):
        pl = T.api.Plan(m, prec, k, r, r + 1)
        pl.execute()
        res = [pl.execute() for _ in range(2)]
        pl.close()
        dm = min(x["device_ms"] for x in res)
        km = min(x["kernel_ms"] for x in res)
        worst = max(worst, dm)
        parts.append(T.torontonian_shard(m, prec, r, P))
        print(f"P={P} rank {r}: device {dm:.3f} ms kernel {km:.3f} ms", flush=True)
    f = T.fold_partials(parts, m)
    if whole is None:
        whole = f["words"]
    print(f"P={P}: max-rank device {worst:.3f} ms -> {2**m.n_modes / (worst * 1e-3):.4e} terms/s; "
          f"fold words {f['words']} identical_to_P1={list(f['words']) == list(whole)}", flush=True)
