"""Generates the committed golden fixtures from the REFERENCE engine.

Run here (where /root/reference exists and oracle/_ref/libtorfp_ref.so is built):

    make -C oracle ref && python tests/golden/make_golden.py [--quick]

Writes
  tests/golden/cfg{1,2,4,5}.gbsa.txt, cfg3_state.gbsa.txt   BASELINE config inputs (lossless)
  tests/golden/reference_values.json                        reference outputs on those inputs
                                                            and on the reference's own test instances
The reference values are produced by the unmodified torfp sources compiled by
oracle/Makefile (torontonian(), torontonian_reference(), select_precision(),
force_width() and the per-mask templates for prefix-class slices).
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
from paper_2009_01177_b200 import workloads as W  # noqa: E402
from paper_2009_01177_b200.matrix import InputMatrix, _upper  # noqa: E402

import numpy as np  # noqa: E402

QUICK = "--quick" in sys.argv
THREADS = os.cpu_count() or 1


def diag_instance(n, a, c=None):
    a00 = np.zeros((n, n), complex)
    a01 = np.zeros((n, n), complex)
    for i in range(n):
        a00[i, i] = a[i]
        if c is not None:
            a01[i, i] = c[i]
    return InputMatrix(n, _upper(a00), _upper(a01))


def full(m, label, prec_list=("128", "256"), fp64=True):
    out = {"label": label, "n": m.n_modes}
    t0 = time.time()
    out["select_precision"] = ref.select_precision(m)
    for w in (128, 256):
        try:
            out[f"force_width_{w}"] = ref.force_width(m, w)
        except ref.RefError as e:
            out[f"force_width_{w}"] = {"error": e.code}
    for p in prec_list:
        try:
            r = ref.torontonian(m, p, THREADS)
            out[f"fixed{p}"] = dict(value=r["value"], raw=str(ref.limbs_to_int(r["raw_limbs"], r["width_bits"])),
                                    frac_bits=r["config"]["frac_bits"], width_bits=r["width_bits"],
                                    counters=r["counters"], wall=r["wall_seconds"])
        except ref.RefError as e:
            out[f"fixed{p}"] = {"error": e.code, "status": e.status, "mask": e.mask, "row": e.row}
    if fp64 and m.n_modes <= 20:
        try:
            out["fp64_reference"] = ref.torontonian_reference(m)
        except ref.RefError as e:
            out["fp64_reference"] = {"error": e.code}
    out["det_i_minus_a"] = ref.det_i_minus_a_float(m)
    print(f"  {label}: {time.time() - t0:.1f}s", flush=True)
    return out


def slices(m, label, k, classes, widths=(128, 256)):
    out = {"label": label, "n": m.n_modes, "k": k, "classes": classes, "widths": {}}
    for w in widths:
        cfg = ref.force_width(m, w)
        res = []
        t0 = time.time()
        for c in classes:
            tot, per, sabs = ref.slice(m, w, cfg["frac_bits"], k, c, c + 1, THREADS)
            res.append(dict(cls=c, raw=str(per[0]), sum_abs=sabs[0]))
        out["widths"][str(w)] = dict(frac_bits=cfg["frac_bits"], classes=res)
        print(f"  {label} slices w={w}: {time.time() - t0:.1f}s", flush=True)
    return out


def main():
    W.write_config_fixtures()
    gold = {"generator": "tests/golden/make_golden.py", "reference": "torfp (oracle/_ref, unmodified sources)",
            "cases": {}}
    C = gold["cases"]

    # --- the reference's own test instances (test_torontonian.cpp, test_precision.cpp)
    for n in range(1, 11):
        C[f"zero_{n}"] = full(diag_instance(n, [0.0] * n), f"zero_{n}", prec_list=("auto",))
    C["half_1"] = full(diag_instance(1, [0.5]), "half_1", prec_list=("auto",))
    C["one_mode"] = full(diag_instance(1, [0.3], [0.1]), "one_mode", prec_list=("auto",))
    C["diag3"] = full(diag_instance(3, [0.1, 0.2, 0.3]), "diag3", prec_list=("auto",))
    C["two_half"] = full(diag_instance(2, [0.5, 0.5]), "two_half", prec_list=("auto",))
    cc = 0.5 - 2.0 ** -20
    C["breakdown6"] = full(diag_instance(6, [0.5] * 6, [cc] * 6), "breakdown6", prec_list=("128", "256"))
    for s in (1, 2, 3):
        C[f"gen10_s{s}"] = full(W.generate_instance(10, 0.16, 0.06, s), f"gen10_s{s}")
    C["gen8_s99"] = full(W.generate_instance(8, 0.16, 0.06, 99), "gen8_s99")
    C["gen10_s321"] = full(W.generate_instance(10, 0.16, 0.06, 321), "gen10_s321")
    C["gen4_s2026"] = full(W.generate_instance(4, 0.16, 0.06, 2026), "gen4_s2026")
    C["gen6_s42"] = full(W.generate_instance(6, 0.16, 0.06, 42), "gen6_s42")
    C["gen12_s7"] = full(W.generate_instance(12, 0.16, 0.06, 7), "gen12_s7")
    C["gen14_s11"] = full(W.generate_instance(14, 0.2, 0.05, 11), "gen14_s11")

    # --- BASELINE configs
    C["cfg1"] = full(W.load_config_instance(1), "cfg1")
    if not QUICK:
        C["cfg2"] = full(W.load_config_instance(2), "cfg2")
    items = range(4 if QUICK else 32)
    C["cfg3_items"] = {}
    for i in items:
        m = W.load_config_instance(3, i)
        C["cfg3_items"][str(i)] = full(m, f"cfg3_{i}", prec_list=("128",) if i >= 8 else ("128", "256"))
    m4 = W.load_config_instance(4)
    C["cfg4"] = {"select_precision": ref.select_precision(m4), "force_width_128": ref.force_width(m4, 128),
                 "force_width_256": ref.force_width(m4, 256), "det_i_minus_a": ref.det_i_minus_a_float(m4)}
    C["cfg4_slices"] = slices(m4, "cfg4", 26, [0, 1, 2, 3, 0x2AAAAAA >> 0, 0x1555555, 0x3FFFFFF, 12345678][: 3 if QUICK else 8])
    m5 = W.load_config_instance(5)
    C["cfg5"] = {"select_precision": ref.select_precision(m5), "force_width_128": ref.force_width(m5, 128),
                 "force_width_256": ref.force_width(m5, 256), "det_i_minus_a": ref.det_i_minus_a_float(m5)}
    C["cfg5_slices"] = slices(m5, "cfg5", 33, [0, 5, (1 << 33) - 1, 0x155555555][: 2 if QUICK else 4])

    with open(os.path.join(HERE, "reference_values.json"), "w") as f:
        json.dump(gold, f, indent=1, sort_keys=True)
    print("wrote reference_values.json")


if __name__ == "__main__":
    main()
