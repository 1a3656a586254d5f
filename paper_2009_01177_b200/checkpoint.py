"""Checkpointed Torontonians: persisted prefix-class partials and resume.

The paper's n = 50 (100 x 100) case is ~6.7 GPU-hours in double-double (profiles/r01_n50_slices_dd.txt);
the reference engine caps N at 40 (torontonian.cpp:153-154) and keeps no intermediate state.  Here a
long evaluation is a sequence of prefix-class slices (tor_torontonian_slice: the classes of the top
`class_bits` reference-mask bits, one device pass each), every finished slice is appended to a
JSON-lines file as an exact record (class range, the unevaluated-sum words, sum |t|, term count:
Python's float repr round-trips doubles exactly), and a restarted run skips the recorded classes.
When every class is recorded the partials fold along the engine's fixed tree (tor_fold_partials):
for class_bits <= 6 the result is bit-identical to an uninterrupted single-device run.

    r = run_checkpointed(m, "128", "n50.ckpt", class_bits=12)   # None until every class is done
"""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from . import api
from .matrix import InputMatrix

FORMAT = "tor-checkpoint-1"


def fingerprint(matrix: InputMatrix, precision, class_bits: int) -> str:
    """Identity of a run: the input's exact doubles, the precision mode and the class split."""
    h = hashlib.sha256()
    h.update(f"{FORMAT}|{matrix.n_modes}|{api._prec(precision)}|{class_bits}|".encode())
    h.update(np.ascontiguousarray(matrix.a00, np.complex128).tobytes())
    h.update(np.ascontiguousarray(matrix.a01, np.complex128).tobytes())
    return h.hexdigest()


def load_records(path: str, fp: str) -> dict[int, dict]:
    """Completed classes of run `fp` in the file (later records of a class win; records of
    other runs and a torn last line from an interrupted write are ignored)."""
    done: dict[int, dict] = {}
    if not os.path.exists(path):
        return done
    with open(path) as f:
        for line in f:
            try:
                rec = json.loads(line)
            except json.JSONDecodeError:
                continue
            if rec.get("format") != FORMAT or rec.get("fingerprint") != fp:
                continue
            done[int(rec["class_lo"])] = rec
    return done


def append_record(path: str, fp: str, part: dict) -> None:
    rec = {"format": FORMAT, "fingerprint": fp, "mode": int(part["mode"]), "class_bits": int(part["class_bits"]),
           "class_lo": int(part["class_lo"]), "class_hi": int(part["class_hi"]),
           "words": [float(w) for w in part["words"]], "sum_abs": float(part["sum_abs"]),
           "term_count": int(part["term_count"])}
    torn = False  # a record torn by an interrupted write: start on a fresh line
    if os.path.exists(path) and os.path.getsize(path) > 0:
        with open(path, "rb") as f:
            f.seek(-1, os.SEEK_END)
            torn = f.read(1) != b"\n"
    with open(path, "a") as f:
        f.write(("\n" if torn else "") + json.dumps(rec) + "\n")
        f.flush()
        os.fsync(f.fileno())


def run_checkpointed(matrix: InputMatrix, precision, path: str, class_bits: int = 6, device: int = 0,
                     max_slices: int | None = None, slice_fn=None) -> dict | None:
    """Evaluate (or resume) Tor(matrix) class by class, persisting each finished class.

    Returns the folded result dict (as torontonian()) once every one of the 2^class_bits classes
    is recorded, else None (e.g. after `max_slices` new classes: a bounded work unit)."""
    if precision in ("auto", api.PREC_AUTO):
        raise api.E.InvalidArgument("precision/range", "checkpointed runs need an explicit precision")
    slice_fn = slice_fn or api.torontonian_slice
    fp = fingerprint(matrix, precision, class_bits)
    done = load_records(path, fp)
    new = 0
    for c in range(1 << class_bits):
        if c in done:
            continue
        if max_slices is not None and new >= max_slices:
            return None
        part = slice_fn(matrix, precision, class_bits, c, c + 1, device=device)
        append_record(path, fp, part)
        done[c] = dict(part)
        new += 1
    parts = [dict(mode=r["mode"], class_bits=r["class_bits"], class_lo=r["class_lo"], class_hi=r["class_hi"],
                  words=tuple(r["words"]), sum_abs=r["sum_abs"], term_count=r["term_count"])
             for _, r in sorted(done.items())]
    return api.fold_partials(parts, matrix)
