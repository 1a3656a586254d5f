"""Reference goldens for the deep Schur-tree paths (multi-level producer DFS, shard-width classes).

Run here (where /root/reference exists and oracle/_ref/libtorfp_ref.so is built):

    make -C oracle ref && python tests/golden/make_golden_deep.py

Input: config 4's instance restricted to its first 30 click modes (n = 30).  The values are
raw fixed-point class sums of the unmodified reference engine (torfp, per-mask templates of
torontonian_partial<W>, torontonian.cpp:72-103) over prefix classes of the top k mask bits
(bit N-1-j = mode j):

  k = 12, class 0xFFF (modes 0..11 all in, 2^18 subsets, the largest determinants' subtree),
         fixed-128 and fixed-256: with a one-job schedule the GPU runs this class as ONE job
         with rjob = 18, i.e. 9 levels of producer DFS;
  k = 6,  classes 0 and 0x2A (2^24 subsets each), fixed-128: shard-width classes, which the
         default n = 30 schedule (c = 18) runs as 4096 jobs each with 3 DFS levels.

And the headline instance itself (config 4, all 32 click modes):

  k = 6,  class 0x15 (2^26 subsets), fixed-128: one of the 64 top-level classes of the measured
         n = 32 double-double run -- the default schedule (c = 18, jobs of 14 modes, five
         producer DFS levels), i.e. exactly what bench.py times and what each rank of a
         multi-GPU run computes (~30 min on 8 cores, as 256 sub-classes of k = 14).

Writes tests/golden/reference_deep.json (~20 min on 8 cores: the k = 6 classes are evaluated as their 64 sub-classes of k = 12 so the harness threads over them).
"""
from __future__ import annotations

import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2009_01177_b200 import matrix as M  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402

THREADS = os.cpu_count() or 1
OUT = os.path.join(HERE, "reference_deep.json")


def n30():
    return M.select_modes(W.load_config_instance(4), list(range(30)))


def slice_case(m, k, cls, widths, split=0):
    """Class `cls` of the top k bits; split > 0 evaluates it as its 2^split sub-classes of the
    top k + split bits (the harness threads over classes) and adds their raw sums -- exact,
    since the reference accumulates in fixed point modulo 2^width."""
    out = {"n": m.n_modes, "k": k, "cls": cls, "widths": {}}
    for w in widths:
        cfg = ref.force_width(m, w)
        t0 = time.time()
        kk, lo, hi = k + split, cls << split, (cls + 1) << split
        tot, per, sabs = ref.slice(m, w, cfg["frac_bits"], kk, lo, hi, THREADS)
        raw = sum(per)
        raw = ((raw + (1 << (w - 1))) % (1 << w)) - (1 << (w - 1))  # modulo 2^w, signed
        out["widths"][str(w)] = dict(frac_bits=cfg["frac_bits"], raw=str(raw), sum_abs=sum(sabs),
                                     seconds=round(time.time() - t0, 1), threads=THREADS,
                                     via=f"{hi - lo} sub-classes of k={kk}" if split else "one class")
        print(f"  n={m.n_modes} k={k} cls={cls:#x} w={w}: {time.time() - t0:.1f}s", flush=True)
    return out


def main():
    m = n30()
    gold = {"generator": "tests/golden/make_golden_deep.py", "reference": "torfp (oracle/_ref, unmodified sources)",
            "instance": "config 4 (tests/golden/cfg4.gbsa.txt), click modes 0..29", "cases": {}}
    if os.path.exists(OUT):
        gold = json.load(open(OUT))
    C = gold["cases"]
    todo = [("n30_k12_fff", 12, 0xFFF, (128, 256), 0), ("n30_k6_00", 6, 0x00, (128,), 6),
            ("n30_k6_2a", 6, 0x2A, (128,), 6), ("n32_k6_15", 6, 0x15, (128,), 8)]
    for name, k, cls, widths, split in todo:
        if name in C:
            continue
        inst = W.load_config_instance(4) if name.startswith("n32") else m
        C[name] = slice_case(inst, k, cls, widths, split)
        with open(OUT, "w") as f:
            json.dump(gold, f, indent=1, sort_keys=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
