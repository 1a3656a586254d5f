"""GPU parity of the deep Schur-tree paths and of the multi-device splits.

The default schedule runs every instance with n <= 27 without producer DFS levels (prefix depth
c = min(18, n - 9)), so these tests force other schedules through the explicit schedule hint of
tor_torontonian_classes (prefix_jobs; replaces round 1's TOR_WANT_JOBS environment knob):
prefix_jobs = 1 makes the whole problem ONE job, i.e. n - Q0 levels of producer DFS (11 at
n = 20), and compare the results with the REFERENCE's outputs (tests/golden/*.json, written
through oracle/_ref):
    DD vs fixed-128 2^-88 sum|t|, QD vs fixed-256 2^-180 sum|t|, fp64 vs fixed-256 2^-44 sum|t|
(the reference's per-worker partial torontonian_partial<W>, torontonian.cpp:72-103).
"""
from __future__ import annotations

import json
import os

import pytest

import paper_2009_01177_b200 as T
from paper_2009_01177_b200 import matrix as M
from paper_2009_01177_b200 import workloads as W
from tests._util import EPS, fixed_value, within, words_value
from tests.test_gpu_parity import GEN_CASES, small_instance

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
MODES = (("128", "fixed128", "dd"), ("256", "fixed256", "qd"), ("fp64", "fixed256", "fp64"))


def whole_with_schedule(m, prec, prefix_jobs):
    """The whole Torontonian as one class (class_bits 0) under a schedule hint."""
    [p] = T.torontonian_classes(m, prec, 0, 0, 1, prefix_jobs=prefix_jobs)
    return p


@pytest.mark.parametrize("prefix_jobs", [1, 8, 64, 4096])
@pytest.mark.parametrize("name", ["cfg2", "gen14_s11", "gen12_s7", "cfg1", "gen10_s1"])
def test_forced_dfs_depth_vs_reference(name, prefix_jobs, golden):
    """Producer DFS depths up to n - Q0 (11 levels for cfg2 at one job) against the
    reference's fixed-128 / fixed-256 values."""
    g = golden[name]
    m = small_instance(name)
    for prec, key, mode in MODES:
        p = whole_with_schedule(m, prec, prefix_jobs)
        want = fixed_value(g[key]["raw"], g[key]["frac_bits"])
        ok, rel = within(words_value(p["words"]), want, p["sum_abs"], mode)
        assert ok, f"{name} {mode} prefix_jobs={prefix_jobs}: err = {rel:.3g} sum|t|"
        assert p["term_count"] == 1 << m.n_modes


@pytest.mark.parametrize("prec", ["128", "256", "fp64"])
def test_schedules_agree_bit_for_bit_only_per_schedule(prec):
    """Same schedule -> bit-identical reruns; the default schedule equals the plain call."""
    m = W.load_config_instance(2)
    a = whole_with_schedule(m, prec, 1)
    b = whole_with_schedule(m, prec, 1)
    assert a["words"] == b["words"] and a["sum_abs"] == b["sum_abs"]
    d = whole_with_schedule(m, prec, 0)
    r = T.torontonian(m, prec)
    assert tuple(d["words"][: len(r["words"])]) == tuple(r["words"])


def _deep():
    path = os.path.join(HERE, "golden", "reference_deep.json")
    if not os.path.exists(path):
        pytest.skip("tests/golden/reference_deep.json not generated")
    return json.load(open(path))["cases"]


def _n30():
    return M.select_modes(W.load_config_instance(4), list(range(30)))


@pytest.mark.parametrize("prefix_jobs", [0, 1, 64])
def test_n30_k12_class_deep_dfs_vs_reference(prefix_jobs):
    """cfg4 restricted to 30 modes, prefix class 0xFFF of the top 12 mask bits (2^18 subsets,
    the largest determinants): prefix_jobs = 1 runs the class as one job with rjob = 18, i.e.
    nine producer DFS levels; the default schedule deepens the prefix instead."""
    case = _deep().get("n30_k12_fff")
    if case is None:
        pytest.skip("n30_k12_fff golden missing")
    m = _n30()
    for prec, mode in (("128", "dd"), ("256", "qd")):
        g = case["widths"]["128" if mode == "dd" else "256"]
        [p] = T.torontonian_classes(m, prec, 12, 0xFFF, 0x1000, prefix_jobs=prefix_jobs)
        want = fixed_value(g["raw"], g["frac_bits"])
        ok, rel = within(words_value(p["words"]), want, p["sum_abs"], mode)
        assert ok, f"{mode} prefix_jobs={prefix_jobs}: err = {rel:.3g} sum|t|"
        assert p["sum_abs"] == pytest.approx(g["sum_abs"], rel=1e-12)
        assert p["term_count"] == 1 << 18


@pytest.mark.parametrize("cls_name,cls", [("n30_k6_00", 0x00), ("n30_k6_2a", 0x2A)])
def test_n30_shard_width_class_vs_reference(cls_name, cls):
    """Shard-width classes (k = 6, 2^24 subsets each) through the default schedule: c = 18,
    rjob = 12, three producer DFS levels -- the configuration an 8-GPU n = 30 run gives
    each rank -- against the reference's fixed-128 class sums."""
    case = _deep().get(cls_name)
    if case is None:
        pytest.skip(f"{cls_name} golden missing")
    m = _n30()
    g = case["widths"]["128"]
    want = fixed_value(g["raw"], g["frac_bits"])
    s = T.torontonian_slice(m, "128", 6, cls, cls + 1)
    ok, rel = within(words_value(s["words"]), want, s["sum_abs"], "dd")
    assert ok, f"slice: err = {rel:.3g} sum|t|"
    [c] = T.torontonian_classes(m, "128", 6, cls, cls + 1)
    assert c["words"] == s["words"]
    q = T.torontonian_slice(m, "256", 6, cls, cls + 1)
    ok, rel = within(words_value(q["words"]), want, q["sum_abs"], "dd")  # fixed-128 bounds the check
    assert ok, f"QD slice vs fixed-128: err = {rel:.3g} sum|t|"


def test_n32_headline_class_vs_reference():
    """The headline instance (config 4, n = 32, double-double), one of its 64 top-level prefix
    classes (k = 6, class 0x15, 2^26 subsets) through the default schedule -- c = 18, jobs of
    14 modes, five producer DFS levels: the pipeline bench.py times and the share of one rank
    of a multi-GPU run -- against the reference's fixed-128 class sum."""
    case = _deep().get("n32_k6_15")
    if case is None:
        pytest.skip("n32_k6_15 golden missing")
    m = W.load_config_instance(4)
    g = case["widths"]["128"]
    want = fixed_value(g["raw"], g["frac_bits"])
    [c] = T.torontonian_classes(m, "128", 6, 0x15, 0x16)
    ok, rel = within(words_value(c["words"]), want, c["sum_abs"], "dd")
    assert ok, f"class partial: err = {rel:.3g} sum|t|"
    assert c["sum_abs"] == pytest.approx(g["sum_abs"], rel=1e-12)
    assert c["term_count"] == 1 << 26
    # the same class inside the whole run's per-class partials (what bench.py's ranks all-gather)
    parts = T.torontonian_classes(m, "128", 6, 0x14, 0x18)
    assert parts[1]["words"] == c["words"]
    # the quad-double pipeline (time-shared areas, jobs of 14 modes) on the same class: the
    # fixed-128 golden bounds the check
    [q] = T.torontonian_classes(m, "256", 6, 0x15, 0x16)
    ok, rel = within(words_value(q["words"]), want, q["sum_abs"], "dd")
    assert ok, f"QD class partial vs fixed-128: err = {rel:.3g} sum|t|"


# ----------------------------------------------------------- class partials / devices --
@pytest.mark.parametrize("prec", ["128", "256", "fp64"])
def test_class_partials_fold_bit_identical(prec):
    """64 per-class partials (any split) fold to the single-device result bit for bit."""
    m = W.load_config_instance(2)
    whole = T.torontonian(m, prec)
    parts = T.torontonian_classes(m, prec, 6, 0, 64)
    assert [p["class_lo"] for p in parts] == list(range(64))
    assert sum(p["term_count"] for p in parts) == 1 << 20
    r = T.fold_partials(parts, m)
    assert r["words"] == whole["words"] and r["sum_abs_terms"] == whole["sum_abs_terms"]
    # uneven contiguous ranges from separate calls (the non-power-of-two device split)
    cuts = [0, 11, 22, 33, 43, 54, 64]
    split = []
    for lo, hi in zip(cuts, cuts[1:]):
        split += T.torontonian_classes(m, prec, 6, lo, hi)
    assert [p["words"] for p in split] == [p["words"] for p in parts]
    # aligned power-of-two blocks of mixed widths fold along the same tree
    blocks = [T.torontonian_slice(m, prec, 6, lo, hi) for lo, hi in ((0, 32), (32, 48), (48, 52), (52, 53),
                                                                      (53, 54), (54, 56), (56, 64))]
    r2 = T.fold_partials(blocks, m)
    assert r2["words"] == whole["words"]


@pytest.mark.parametrize("ndev", [2, 3, 5, 6, 7, 8])
def test_device_lists_any_count_bit_identical(ndev):
    """tor_torontonian over `ndev` listed devices (here all device 0: one host thread each)
    uses every device and matches one device bit for bit (no power-of-two truncation)."""
    m = W.load_config_instance(2)
    for prec in ("128", "256", "fp64"):
        one = T.torontonian(m, prec)
        r = T.torontonian(m, prec, devices=[0] * ndev)
        assert r["devices"] == ndev
        assert r["words"] == one["words"] and r["sum_abs_terms"] == one["sum_abs_terms"]


@pytest.mark.parametrize("n", [1, 2, 10, 14])
def test_device_lists_small_instances(n):
    """Instances without 6 prefix levels run on the first device (round-1 advisor: n <= 2
    with 4/8 devices read past the triangle; n = 10 with 4 devices changed arithmetic)."""
    m = W.generate_instance(n, 0.16, 0.06, 5)
    for prec in ("128", "256", "fp64"):
        one = T.torontonian(m, prec)
        for ndev in (2, 4, 8):
            r = T.torontonian(m, prec, devices=[0] * ndev)
            assert r["words"] == one["words"]
            assert r["devices"] == 1 if n <= 10 else r["devices"] in (1, ndev)


def test_fold_rejects_incomplete_or_mixed_partials():
    m = W.load_config_instance(2)
    parts = [T.torontonian_shard(m, "128", r, 4) for r in range(4)]
    T.fold_partials(parts, m)
    with pytest.raises(T.InvalidArgument):
        T.fold_partials(parts[:3], m)          # a rank missing at the end
    with pytest.raises(T.InvalidArgument):
        T.fold_partials(parts[1:], m)          # ... at the start
    with pytest.raises(T.InvalidArgument):
        T.fold_partials(parts[:1] + parts[2:], m)  # ... in the middle (not contiguous)
    q = T.torontonian_shard(m, "256", 1, 4)
    with pytest.raises(T.InvalidArgument):
        T.fold_partials([parts[0], q, parts[2], parts[3]], m)  # mixed modes
    bad = T.torontonian_slice(m, "128", 2, 1, 3)              # [1,3): not aligned
    with pytest.raises(T.InvalidArgument):
        T.fold_partials([parts[0], bad, parts[3]], m)


def test_invalid_precisions_rejected():
    m = W.load_config_instance(2)
    for bad in (0, 4, 5, 17, -1):
        with pytest.raises(T.InvalidArgument):
            T.api._check(*_raw_slice(m, bad))


def _raw_slice(m, prec):
    import ctypes as C
    inp = T.api._In(m)
    p = T.api.TorPartial()
    err = T.api.TorError()
    st = T.api.lib().tor_torontonian_slice(C.byref(inp.s), prec, 1, 0, 1, 0, C.byref(p), C.byref(err))
    return st, err
