"""Checkpointed runs (paper_2009_01177_b200.checkpoint): persisted class partials and resume.

CPU: the record file logic with a stub slice function (exact fixed-point class sums from the
oracle as DD words), the fold through tor_fold_partials (host code).  GPU: an interrupted and
resumed run folds bit-identically to the uninterrupted single-device result."""
from __future__ import annotations

import json
from fractions import Fraction

import pytest

import paper_2009_01177_b200 as T
from paper_2009_01177_b200 import api, checkpoint
from paper_2009_01177_b200 import workloads as W
from tests._util import fixed_value


def _oracle_slice_fn(calls):
    from oracle import port as P

    def fn(m, precision, k, lo, hi, device=0):
        calls.append((k, lo, hi))
        f = T.force_width(m, 128)["frac_bits"]
        tot, per, sabs = P.slice(m, 128, f, k, lo, hi, threads=2)
        x = Fraction(tot, 1 << f)
        hi_w = float(x)
        return dict(mode=api.PREC_DD, class_bits=k, class_lo=lo, class_hi=hi,
                    words=(hi_w, float(x - Fraction(hi_w)), 0.0, 0.0), sum_abs=sum(sabs),
                    term_count=(hi - lo) << (m.n_modes - k))
    return fn


def test_resume_skips_recorded_classes(tmp_path, golden):
    m = W.load_config_instance(1)  # n = 16
    path = str(tmp_path / "run.ckpt")
    calls = []
    fn = _oracle_slice_fn(calls)
    assert checkpoint.run_checkpointed(m, "128", path, class_bits=3, max_slices=3, slice_fn=fn) is None
    assert [c[1] for c in calls] == [0, 1, 2]
    with open(path, "a") as f:
        f.write('{"format": "tor-checkpoint-1", "fingerprint": "torn')  # an interrupted write
    r = checkpoint.run_checkpointed(m, "128", path, class_bits=3, slice_fn=fn)
    assert [c[1] for c in calls] == [0, 1, 2, 3, 4, 5, 6, 7]  # resumed at class 3
    g = golden["cfg1"]["fixed128"]
    got = sum((Fraction(w) for w in r["words"]), Fraction(0))
    assert abs(float(got - fixed_value(g["raw"], g["frac_bits"]))) <= 2.0 ** -100 * r["sum_abs_terms"]
    # a finished file folds again without any new slice; other runs' records are ignored
    m2 = W.generate_instance(16, 0.16, 0.06, 1)
    assert checkpoint.fingerprint(m2, "128", 3) != checkpoint.fingerprint(m, "128", 3)
    r2 = checkpoint.run_checkpointed(m, "128", path, class_bits=3, slice_fn=fn)
    assert len(calls) == 8 and r2["words"] == r["words"]
    recs = [json.loads(x) for x in open(path) if x.startswith('{"format": "tor-checkpoint-1", "fingerprint": "') and
            x.rstrip().endswith("}")]
    assert sorted(rec["class_lo"] for rec in recs) == list(range(8))


def test_auto_precision_rejected(tmp_path):
    with pytest.raises(T.InvalidArgument):
        checkpoint.run_checkpointed(W.load_config_instance(1), "auto", str(tmp_path / "x"))


@pytest.mark.gpu
@pytest.mark.parametrize("prec", ["128", "256"])
def test_interrupted_run_folds_bit_identically(tmp_path, prec):
    m = W.load_config_instance(2)  # n = 20
    path = str(tmp_path / "cfg2.ckpt")
    assert checkpoint.run_checkpointed(m, prec, path, class_bits=4, max_slices=5) is None
    assert checkpoint.run_checkpointed(m, prec, path, class_bits=4, max_slices=6) is None
    r = checkpoint.run_checkpointed(m, prec, path, class_bits=4)
    whole = T.torontonian(m, prec)
    assert r["words"] == whole["words"] and r["sum_abs_terms"] == whole["sum_abs_terms"]
    assert r["raw_limbs"] == whole["raw_limbs"]
