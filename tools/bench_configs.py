"""Runs every BASELINE.json config once on the GPU and prints one JSON record per config.

cfg1 n=16 fp64 | cfg2 n=20 DD | cfg3 4096 x n=16 fp64 + DD (batch) | cfg4 n=32 QD (+ DD headline) |
cfg5 n=40 DD with the adaptive bound check (precision "auto").  Device times are CUDA-event
times of the engine pipeline (inputs resident via tor_plan where applicable).
"""
from __future__ import annotations

import json
import sys
import time

sys.path.insert(0, ".")
import paper_2009_01177_b200 as T  # noqa: E402
from paper_2009_01177_b200 import workloads as W  # noqa: E402


def run_one(cfg, prec, reps=2):
    m = W.load_config_instance(cfg)
    T.torontonian(m, prec)
    best = None
    for _ in range(reps):
        t0 = time.time()
        r = T.torontonian(m, prec)
        r["wall"] = time.time() - t0
        if best is None or r["device_ms"] < best["device_ms"]:
            best = r
    return m, best


def rec(cfg, prec, r, n):
    return {"config": cfg, "n": n, "precision": prec, "mode": r["mode"], "value": r["value"],
            "words": list(r["words"]), "device_ms": r["device_ms"], "kernel_ms": r["kernel_ms"],
            "wall_s": r["wall"], "terms_per_s": r["term_count"] / (r["device_ms"] * 1e-3),
            "sum_abs_terms": r["sum_abs_terms"], "cancellation_bits": r["cancellation_bits"],
            "bits_left": r["bits_left"], "escalated": r["escalated"], "config_sel": r["config"]}


def main():
    which = sys.argv[1].split(",") if len(sys.argv) > 1 else ["1", "2", "3", "4dd", "4qd", "5"]
    for w in which:
        if w == "1":
            m, r = run_one(1, "fp64")
            print(json.dumps(rec(1, "fp64", r, m.n_modes)), flush=True)
        elif w == "2":
            m, r = run_one(2, "128")
            print(json.dumps(rec(2, "128", r, m.n_modes)), flush=True)
        elif w == "3":
            ms = W.load_cfg3_batch(4096)
            for prec in ("fp64", "128"):
                T.torontonian_batch(ms[:64], prec)
                t0 = time.time()
                rs = T.torontonian_batch(ms, prec)
                wall = time.time() - t0
                dev = rs[0]["device_ms"]
                print(json.dumps({"config": 3, "n": 16, "items": len(ms), "precision": prec, "device_ms": dev,
                                  "wall_s": wall, "terms_per_s": len(ms) * (1 << 16) / (dev * 1e-3),
                                  "item0_value": rs[0]["value"], "item0_words": list(rs[0]["words"])}), flush=True)
        elif w == "4dd":
            m, r = run_one(4, "128")
            print(json.dumps(rec(4, "128", r, m.n_modes)), flush=True)
        elif w == "4qd":
            m, r = run_one(4, "256", reps=1)
            print(json.dumps(rec(4, "256", r, m.n_modes)), flush=True)
        elif w == "5":
            m = W.load_config_instance(5)
            t0 = time.time()
            r = T.torontonian(m, "auto")
            r["wall"] = time.time() - t0
            print(json.dumps(rec(5, "auto", r, m.n_modes)), flush=True)


if __name__ == "__main__":
    main()
