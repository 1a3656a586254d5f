"""QD engine stress (development aid): sub-instances of config 4 with n = 9..27 modes, QD twice
(bit-identical) and against DD (within 2^-90 sum|t|); device-list runs of 2 and 3 shards."""
import sys
sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import matrix as M  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402
full = W.load_config_instance(4)
bad = 0
for n in range(9, 28):
    m = M.select_modes(full, list(range(n)))
    a = T.torontonian(m, "256")
    b = T.torontonian(m, "256")
    d = T.torontonian(m, "128")
    same = a["words"] == b["words"]
    err = abs(a["value"] - d["value"])
    ok = same and err <= 2.0 ** -90 * a["sum_abs_terms"]
    extra = ""
    if n >= 17:
        c = T.torontonian(m, "256", devices=[0, 0, 0])
        ok = ok and c["words"] == a["words"]
        extra = f" devices3_identical={c['words'] == a['words']}"
    bad += not ok
    print(f"n={n}: qd={a['value']:.17e} repeat_identical={same} |qd-dd|/sum|t|={err / a['sum_abs_terms']:.2e}{extra} "
          f"kernel {a['kernel_ms']:.3f} ms {'ok' if ok else 'FAIL'}", flush=True)
print("failures:", bad)
sys.exit(1 if bad else 0)
