"""Kernel time of one whole Torontonian under different prefix-job counts (schedule hint of
tor_torontonian_classes): python tools/sched_probe.py CFG PREC [MODES] -- JOBS..."""
import sys
sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import matrix as M  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402
args = sys.argv[1:]
k = args.index("--")
cfg, prec = int(args[0]), args[1]
m = W.load_config_instance(cfg)
if k > 2:
    m = M.select_modes(m, list(range(int(args[2]))))
for jobs in [int(x) for x in args[k + 1:]]:
    T.torontonian_classes(m, prec, 0, 0, 1, prefix_jobs=jobs)
    [p] = T.torontonian_classes(m, prec, 0, 0, 1, prefix_jobs=jobs)
    print(jobs, {x: p[x] for x in p if x in ("kernel_ms", "device_ms", "words")}, flush=True)
