"""GPU parity: the CUDA engine (through the C ABI) vs the reference's own outputs.

Golden values come from the unmodified reference engine (tests/golden/reference_values.json,
written by tests/golden/make_golden.py through oracle/_ref).  Tolerances are absolute,
against sum |terms| because the alternating sum cancels:
    fp64 vs torontonian_reference  2^-44 sum|t|
    DD   vs fixed-128              2^-88 sum|t|
    QD   vs fixed-256              2^-180 sum|t|
plus |rel| <= 1e-3 (b_sgn = 3 digits) wherever the mode keeps the digits.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2009_01177_b200 as T
from paper_2009_01177_b200 import workloads as W
from paper_2009_01177_b200.matrix import InputMatrix, _upper
from tests._util import EPS, fixed_value, within, words_value

pytestmark = pytest.mark.gpu


def diag_instance(n, a, c=None):
    a00 = np.zeros((n, n), complex)
    a01 = np.zeros((n, n), complex)
    for i in range(n):
        a00[i, i] = a[i]
        if c is not None:
            a01[i, i] = c[i]
    return InputMatrix(n, _upper(a00), _upper(a01))


def small_instance(name):
    if name.startswith("zero_"):
        n = int(name.split("_")[1])
        return diag_instance(n, [0.0] * n)
    fixed = {
        "half_1": lambda: diag_instance(1, [0.5]),
        "one_mode": lambda: diag_instance(1, [0.3], [0.1]),
        "diag3": lambda: diag_instance(3, [0.1, 0.2, 0.3]),
        "two_half": lambda: diag_instance(2, [0.5, 0.5]),
        "breakdown6": lambda: diag_instance(6, [0.5] * 6, [0.5 - 2.0 ** -20] * 6),
        "gen10_s1": lambda: W.generate_instance(10, 0.16, 0.06, 1),
        "gen10_s2": lambda: W.generate_instance(10, 0.16, 0.06, 2),
        "gen10_s3": lambda: W.generate_instance(10, 0.16, 0.06, 3),
        "gen8_s99": lambda: W.generate_instance(8, 0.16, 0.06, 99),
        "gen10_s321": lambda: W.generate_instance(10, 0.16, 0.06, 321),
        "gen4_s2026": lambda: W.generate_instance(4, 0.16, 0.06, 2026),
        "gen6_s42": lambda: W.generate_instance(6, 0.16, 0.06, 42),
        "gen12_s7": lambda: W.generate_instance(12, 0.16, 0.06, 7),
        "gen14_s11": lambda: W.generate_instance(14, 0.2, 0.05, 11),
        "cfg1": lambda: W.load_config_instance(1),
        "cfg2": lambda: W.load_config_instance(2),
    }
    return fixed[name]()


GEN_CASES = ["gen10_s1", "gen10_s2", "gen10_s3", "gen8_s99", "gen10_s321", "gen4_s2026", "gen6_s42",
             "gen12_s7", "gen14_s11", "cfg1", "cfg2"]


@pytest.mark.parametrize("n", range(1, 11))
def test_zero_matrix_exactly_zero(n, golden):
    """test_torontonian.cpp:49-61: Tor(0) = 0 limb-exact, term_count = 2^N."""
    m = small_instance(f"zero_{n}")
    for prec in ("auto", "128", "256", "fp64"):
        r = T.torontonian(m, prec)
        assert r["value"] == 0.0
        assert all(w == 0.0 for w in r["words"])
        assert r["raw_limbs"] == (0, 0, 0, 0)
        assert r["term_count"] == 1 << n
    assert T.torontonian_reference(m) == 0.0
    assert golden[f"zero_{n}"]["fixedauto"]["raw"] == "0"


def test_closed_forms():
    """test_torontonian.cpp:63-81 single-mode and diagonal closed forms, at DD accuracy."""
    cases = [
        (small_instance("half_1"), 1.0),
        (small_instance("one_mode"), 1.0 / math.sqrt(0.7 * 0.7 - 0.01) - 1.0),
        (small_instance("diag3"), (0.1 / 0.9) * (0.2 / 0.8) * (0.3 / 0.7)),
        (small_instance("two_half"), 1.0),
    ]
    for m, want in cases:
        for prec in ("auto", "128", "256"):
            assert T.torontonian(m, prec)["value"] == pytest.approx(want, rel=1e-12)
        assert T.torontonian_reference(m) == pytest.approx(want, rel=1e-12)


@pytest.mark.parametrize("name", GEN_CASES)
def test_modes_vs_reference(name, golden):
    g = golden[name]
    m = small_instance(name)
    # DD vs reference fixed-128, QD vs fixed-256 (same inputs)
    for prec, key, mode in (("128", "fixed128", "dd"), ("256", "fixed256", "qd")):
        r = T.torontonian(m, prec)
        want = fixed_value(g[key]["raw"], g[key]["frac_bits"])
        ok, rel = within(words_value(r["words"]), want, r["sum_abs_terms"], mode)
        assert ok, f"{name} {mode}: err = {rel:.3g} sum|t| (eps {EPS[mode]:.3g})"
        assert abs(r["value"] - float(want)) <= 1e-3 * abs(float(want))
        assert r["config"]["frac_bits"] == g[key]["frac_bits"]
        assert r["counters"] == g[key]["counters"]
    # fp64 mode vs the reference fp64 oracle (both accurate to ~2^-44 sum|t| only)
    if isinstance(g.get("fp64_reference"), float):
        v = T.torontonian_reference(m)
        r = T.torontonian(m, "fp64")
        ok, rel = within(v, g["fp64_reference"], r["sum_abs_terms"], "fp64")
        assert ok, f"{name} fp64: err = {rel:.3g} sum|t|"
        # and the GPU fp64 vs the exact (fixed-256) value
        ok2, rel2 = within(v, fixed_value(g["fixed256"]["raw"], g["fixed256"]["frac_bits"]), r["sum_abs_terms"], "fp64")
        assert ok2, f"{name} fp64 vs fixed256: {rel2:.3g}"


@pytest.mark.parametrize("name", GEN_CASES)
def test_auto_matches_reference_selection(name, golden):
    g = golden[name]
    m = small_instance(name)
    r = T.torontonian(m, "auto")
    sel = g["select_precision"]
    assert r["config"]["width_bits"] == sel["width_bits"]
    assert r["config"]["frac_bits"] == sel["frac_bits"]
    assert r["width_bits"] == sel["width_bits"] or r["escalated"]


def test_breakdown_instance_succeeds_in_floating_words(golden):
    """test_torontonian.cpp:218-244: fixed-128 breaks down (fraction bits exhausted);
    DD/QD keep relative precision and reproduce the closed form."""
    g = golden["breakdown6"]
    assert g["fixed128"]["error"] == "linalg/breakdown"
    m = small_instance("breakdown6")
    c = 0.5 - 2.0 ** -20
    want = (1.0 / math.sqrt(0.25 - c * c) - 1.0) ** 6
    for prec in ("128", "256"):
        r = T.torontonian(m, prec)
        assert abs(r["value"] - want) / want < 1e-9
    # the reference's own 256-bit value is only good to ~3e-5 here
    assert abs(g["fixed256"]["value"] - want) / want < 1e-3


def test_cfg3_items(golden):
    items = golden["cfg3_items"]
    ms = [W.load_config_instance(3, int(i)) for i in sorted(items, key=int)]
    batch_dd = T.torontonian_batch(ms, "128")
    batch_64 = T.torontonian_batch(ms, "fp64")
    for k, (i, g) in enumerate(sorted(items.items(), key=lambda kv: int(kv[0]))):
        want = fixed_value(g["fixed128"]["raw"], g["fixed128"]["frac_bits"])
        ok, rel = within(words_value(batch_dd[k]["words"]), want, batch_dd[k]["sum_abs_terms"], "dd")
        assert ok, f"cfg3 item {i}: {rel:.3g}"
        single = T.torontonian(ms[k], "128")
        assert single["words"] == batch_dd[k]["words"], "batch must be bit-identical to single runs"
        ok, rel = within(words_value(batch_64[k]["words"]), want, batch_64[k]["sum_abs_terms"], "fp64")
        assert ok, f"cfg3 item {i} fp64: {rel:.3g}"


@pytest.mark.parametrize("cfg", ["cfg4_slices", "cfg5_slices"])
def test_large_n_slices(cfg, golden):
    """n=32 / 40: prefix-class slices through the reference's per-mask templates."""
    g = golden[cfg]
    m = W.load_config_instance(4 if cfg == "cfg4_slices" else 5)
    k = g["k"]
    for width, mode, prec in (("128", "dd", "128"), ("256", "qd", "256")):
        if width not in g["widths"]:
            continue
        gw = g["widths"][width]
        for c in gw["classes"]:
            p = T.torontonian_slice(m, prec, k, c["cls"], c["cls"] + 1)
            want = fixed_value(c["raw"], gw["frac_bits"])
            ok, rel = within(words_value(p["words"]), want, c["sum_abs"], mode)
            assert ok, f"{cfg} class {c['cls']:#x} {mode}: {rel:.3g} sum|t|"
            assert p["sum_abs"] == pytest.approx(c["sum_abs"], rel=1e-9)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_shards_fold_bit_identical(world):
    m = W.load_config_instance(2)
    for prec in ("128", "256", "fp64"):
        whole = T.torontonian(m, prec)
        parts = [T.torontonian_shard(m, prec, r, world) for r in range(world)]
        folded = T.fold_partials(parts, m)
        assert folded["words"] == whole["words"]
        assert folded["sum_abs_terms"] == whole["sum_abs_terms"]


def test_shards_fold_bit_identical_n32_dd():
    # the headline configuration: 1/2/4/8 shards of the n=32 DD Torontonian fold to the
    # identical words (the prefix depth does not depend on the shard's class range)
    m = W.load_config_instance(4)
    whole = T.torontonian(m, "128")
    for world in (2, 4, 8):
        parts = [T.torontonian_shard(m, "128", r, world) for r in range(world)]
        folded = T.fold_partials(parts, m)
        assert folded["words"] == whole["words"], world
        assert folded["sum_abs_terms"] == whole["sum_abs_terms"], world


def test_determinism_reruns():
    m = W.load_config_instance(1)
    a = T.torontonian(m, "128")
    b = T.torontonian(m, "128")
    assert a["words"] == b["words"]


def test_input_validation():
    big = diag_instance(41, [0.0] * 41)
    with pytest.raises(T.InvalidArgument):
        T.torontonian(big)
    wide = diag_instance(21, [0.0] * 21)
    with pytest.raises(T.InvalidArgument):
        T.torontonian_reference(wide)
    skew = diag_instance(2, [0.2, 0.2])
    skew.a00[0] = 0.2 + 0.05j
    with pytest.raises(T.TorfpError) as e:
        T.torontonian(skew)
    assert e.value.code == "torontonian/symmetry"
    indef = diag_instance(1, [0.5], [0.7])
    with pytest.raises(T.PrecisionError):
        T.torontonian(indef)


def test_indefinite_breakdown_reports_mask():
    """A non-positive pivot in working precision raises linalg/breakdown with a mask."""
    m = diag_instance(3, [0.1, 0.5, 0.1], [0.0, 0.7, 0.0])
    with pytest.raises((T.BreakdownError, T.PrecisionError)):
        T.torontonian(m, "128")


@pytest.mark.parametrize("prec", ["fp64", "128", "256"])
def test_breakdown_mask_at_every_tree_level(prec):
    """Two indefinite modes in an n = 24 instance (det(I - O) > 0 overall): the engine reports
    a single-mode subset (smallest failing mask, one of its two pivot rows) whichever tree level
    evaluates those modes -- prefix levels, producer DFS / fan-out, or the consumers' lane
    subtrees, where the key is kept per thread and published once."""
    n = 24
    masks, rows = [], set()
    for k in (0, 4, 9, 14, 22):
        a = [0.1] * n
        c = [0.05] * n
        for j in (k, k + 1):
            a[j], c[j] = 0.5, 0.7  # det of I - O_{j} = 0.25 - 0.49 < 0
        with pytest.raises(T.BreakdownError) as e:
            T.torontonian(diag_instance(n, a, c), prec)
        assert bin(e.value.subset_mask).count("1") == 1, (k, e.value.subset_mask)
        rows.add(e.value.pivot_row)
        masks.append(e.value.subset_mask)
    assert len(set(masks)) == len(masks)
    assert len(rows) == 1 and rows <= {0, 1}, rows  # the same pivot row of a one-mode subset


@pytest.mark.parametrize("prec", ["fp64", "128", "256"])
def test_negative_definite_block_breaks_down_at_every_level(prec):
    """A mode whose 2x2 block of I - O is negative definite (det > 0, so det(I - O) > 0 and
    the one-mode Torontonian term is finite) must still break down at the first pivot, as the
    reference's Cholesky does -- including when that mode is the last one eliminated (the
    leaf term, which otherwise needs only the determinant)."""
    n = 24
    masks = []
    for k in (0, 4, 9, 14, 22, 23):
        a = [0.1] * n
        c = [0.05] * n
        a[k], c[k] = 1.5, 0.1  # eigenvalues of the block: -0.6, -0.4
        with pytest.raises(T.BreakdownError) as e:
            T.torontonian(diag_instance(n, a, c), prec)
        assert bin(e.value.subset_mask).count("1") == 1, (k, e.value.subset_mask)
        assert e.value.pivot_row == 0, (k, e.value.pivot_row)
        masks.append(e.value.subset_mask)
    assert len(set(masks)) == len(masks)


def test_probabilities():
    """test_torontonian.cpp:246-268."""
    a = diag_instance(1, [0.3], [0.1])
    det = 0.7 * 0.7 - 0.01
    p1 = T.probability(a, 1)
    p0 = T.probability(a, 0)
    assert p1 == pytest.approx(1.0 - math.sqrt(det), rel=1e-12)
    assert p0 == pytest.approx(math.sqrt(det), rel=1e-12)
    m = W.generate_instance(4, 0.16, 0.06, 1234)
    assert sum(T.probability_reference(m, b) for b in range(16)) == pytest.approx(1.0, rel=1e-9)


# ---------------------------------------------------- exact fixed-point mode ----
FIXED_CASES = ["gen10_s1", "gen10_s2", "gen10_s3", "gen8_s99", "gen10_s321", "gen4_s2026", "gen6_s42",
               "gen12_s7", "gen14_s11", "cfg1", "half_1", "one_mode", "diag3", "two_half", "zero_7"]


@pytest.mark.parametrize("name", FIXED_CASES)
def test_fixed_point_mode_limb_exact(name, golden):
    """GPU exact fixed-point validation mode: the reference's algorithm on the integer
    pipes reproduces the reference's raw accumulator limbs exactly."""
    g = golden[name]
    m = small_instance(name)
    for p, key in (("fixed128", "fixed128"), ("fixed256", "fixed256")):
        r = T.torontonian(m, p)
        ref = g.get(key) or g.get("fixedauto")
        if key not in g and r["width_bits"] != 128:
            continue
        assert r["config"]["frac_bits"] == ref["frac_bits"]
        from oracle.ref import limbs_to_int
        assert limbs_to_int(r["raw_limbs"], r["width_bits"]) == int(ref["raw"]), f"{name} {p}"
        assert r["value"] == ref["value"]


def test_fixed_point_mode_breakdown_like_reference(golden):
    m = small_instance("breakdown6")
    with pytest.raises(T.BreakdownError) as e:
        T.torontonian(m, "fixed128")
    assert e.value.code == "linalg/breakdown"
    r = T.torontonian(m, "fixed256")
    from oracle.ref import limbs_to_int
    assert limbs_to_int(r["raw_limbs"], 256) == int(golden["breakdown6"]["fixed256"]["raw"])


def test_grid_scaling_for_large_diagonals():
    """DD states use a fixed-exponent leading word (needs max R_kk < 15); larger inputs
    are scaled by an exact power of two and every term is scaled back by 2^(-s|Z|)."""
    for n, a, c in ((3, -20.0, 0.0), (10, -40.0, 5.0), (12, 0.1, 0.0)):
        m = diag_instance(n, [a] * n, [c] * n)
        want = (1.0 / math.sqrt((1 - a) ** 2 - c * c) - 1.0) ** n
        for prec in ("128", "256", "fp64"):
            r = T.torontonian(m, prec)
            assert r["value"] == pytest.approx(want, rel=1e-11), (n, a, prec)


@pytest.mark.parametrize("n", [24, 28])
def test_full_pipeline_dd_vs_qd(n):
    """The full device pipeline (prefix levels, warp DFS, fan-out, TMEM lane handoff,
    grid-DD Schur updates) at n where every stage runs: DD vs the GPU's own QD (which
    agrees with the reference's fixed-256 at 2^-180 sum|t| on every golden case)."""
    from paper_2009_01177_b200.matrix import select_modes
    m = select_modes(W.load_config_instance(5), list(range(n)))
    dd = T.torontonian(m, "128")
    q = T.torontonian(m, "256")
    ok, rel = within(words_value(dd["words"]), words_value(q["words"]), q["sum_abs_terms"], "dd")
    assert ok, f"n={n}: DD vs QD {rel:.3g} sum|t|"
    assert rel < 2.0 ** -100
    assert abs(dd["sum_abs_terms"] - q["sum_abs_terms"]) <= 1e-12 * q["sum_abs_terms"]


@pytest.mark.parametrize("prec,mode", [("128", "dd"), ("256", "qd"), ("fp64", "fp64")])
def test_uneven_class_ranges(prec, mode):
    # class ranges that are not aligned powers of two (ragged prefix-level ranges, a
    # fixed-order fold over a non-power-of-two job count): the pieces add up to the whole
    m = W.load_config_instance(2)
    whole = T.torontonian(m, prec)
    for k, cuts in ((3, (0, 3, 8)), (5, (0, 1, 7, 19, 32)), (9, (0, 100, 301, 512))):
        parts = [T.torontonian_slice(m, prec, k, a, b) for a, b in zip(cuts, cuts[1:])]
        total = sum((words_value(p["words"]) for p in parts), start=words_value([0.0]))
        sum_abs = sum(p["sum_abs"] for p in parts)
        assert sum_abs == pytest.approx(whole["sum_abs_terms"], rel=1e-12)
        ok, rel = within(total, words_value(whole["words"]), whole["sum_abs_terms"], mode)
        assert ok, f"k={k} cuts={cuts}: {rel:.3g} sum|t|"


def _cfg5_extended(n):
    # config 5's m = 100 state, its 40 click modes plus the lowest unused ones
    from paper_2009_01177_b200.matrix import select_modes
    sel = set(W.click_set(5))
    extra = [j for j in range(100) if j not in sel][: n - 40]
    return select_modes(W.full_state(5), sorted(sel | set(extra)))


def test_slices_beyond_n40():
    # the reference's torontonian() takes N <= 40; slices / shards go to N = 50 (the paper's
    # 100 x 100 case) as checkpointable class ranges.  n = 44: one class at k = 22 (2^22
    # subsets) in DD and QD, and its refinement into two classes at k = 23.
    m = _cfg5_extended(44)
    with pytest.raises(T.InvalidArgument):
        T.torontonian(m, "128")
    k, cls = 22, 0x2a5a5
    dd = T.torontonian_slice(m, "128", k, cls, cls + 1)
    qd = T.torontonian_slice(m, "256", k, cls, cls + 1)
    ok, rel = within(words_value(dd["words"]), words_value(qd["words"]), qd["sum_abs"], "dd")
    assert ok, f"DD vs QD {rel:.3g} sum|t|"
    assert dd["term_count"] == 1 << (44 - k)
    halves = [T.torontonian_slice(m, "256", k + 1, 2 * cls + h, 2 * cls + h + 1) for h in (0, 1)]
    tot = words_value(halves[0]["words"]) + words_value(halves[1]["words"])
    ok, rel = within(tot, words_value(qd["words"]), qd["sum_abs"], "qd")
    assert ok, f"refinement {rel:.3g} sum|t|"
    # a whole-range slice at n = 50 is accepted and sized by class range (shard of 2^14)
    m50 = _cfg5_extended(50)
    p = T.torontonian_slice(m50, "128", 30, 12345, 12346)
    assert p["term_count"] == 1 << 20 and p["sum_abs"] > 0
    with pytest.raises(T.InvalidArgument):
        T.torontonian_slice(_cfg5_extended(51), "128", 30, 0, 1)


def test_batch_beyond_grid_y_limit():
    # 70000 instances: the per-instance fold passes run in chunks of 65535 grid rows
    base = [W.generate_instance(12, 0.16, 0.06, s) for s in range(1, 9)]
    ms = [base[i % 8] for i in range(70000)]
    rs = T.torontonian_batch(ms, "128")
    singles = [T.torontonian(b, "128") for b in base]
    for i in (0, 7, 65534, 65535, 65536, 69999):
        want = singles[i % 8]
        ok, rel = within(words_value(rs[i]["words"]), words_value(want["words"]), want["sum_abs_terms"], "dd")
        assert ok, f"item {i}: {rel:.3g} sum|t|"


def test_headline_n32_dd_vs_qd():
    # the headline Torontonian itself (config 4's input, n = 32, 2^32 subsets): DD against
    # the GPU's own QD, the full-size check the reference cannot run (2.4e5 s in fixed-128)
    m = W.load_config_instance(4)
    dd = T.torontonian(m, "128")
    q = T.torontonian(m, "256")
    ok, rel = within(words_value(dd["words"]), words_value(q["words"]), q["sum_abs_terms"], "dd")
    assert ok, f"DD vs QD {rel:.3g} sum|t|"
    assert rel < 2.0 ** -100
    assert abs(float(words_value(dd["words"]) / words_value(q["words"])) - 1.0) < 1e-12


@pytest.mark.parametrize("prec", ["fp64", "128", "256"])
def test_plan_resident_repeats(prec):
    # tor_plan_*: inputs uploaded once, execute() reruns the whole device pipeline; every
    # rerun gives the same words as the one-shot call, and a sharded plan its shard's words
    m = W.load_config_instance(2)
    whole = T.torontonian(m, prec)
    pl = T.api.Plan(m, prec)
    try:
        for _ in range(3):
            r = pl.execute()
            assert r["words"] == whole["words"]
            assert r["kernel_launches"] > 0 and r["device_ms"] > 0
    finally:
        pl.close()
    shard = T.torontonian_shard(m, prec, 1, 4)
    ps = T.api.Plan(m, prec, 2, 1, 2)
    try:
        assert ps.execute()["words"][: len(shard["words"])] == shard["words"][: len(ps.execute()["words"])]
    finally:
        ps.close()


def test_batch_auto_mixed_widths():
    # batch AUTO selects the width per instance like tor_torontonian: the near-singular
    # instance needs 256 bits (QD sub-batch), the others 128 (DD sub-batch)
    hard = diag_instance(6, [0.5] * 6, [0.5 - 2.0 ** -20] * 6)
    ms = [W.generate_instance(6, 0.16, 0.06, s) for s in (1, 2)] + [hard] + [W.generate_instance(6, 0.16, 0.06, 3)]
    rs = T.torontonian_batch(ms, "auto")
    assert [r["mode"] for r in rs] == ["dd", "dd", "qd", "dd"]
    for m, r in zip(ms, rs):
        single = T.torontonian(m, "auto")
        assert r["mode"] == single["mode"] and r["config"] == single["config"]
        ok, rel = within(words_value(r["words"]), words_value(single["words"]), single["sum_abs_terms"], r["mode"])
        assert ok, rel
    closed = (1.0 / math.sqrt((1 - 0.5) ** 2 - (0.5 - 2.0 ** -20) ** 2) - 1.0) ** 6
    assert abs(rs[2]["value"] / closed - 1) < 1e-9


def test_probability_beyond_64_modes():
    # p(S) on config 3's m = 100 state (the reference's u64 ClickPattern cannot address it):
    # the mode-list entry point equals Tor(O_S) sqrt(det(I - O)) of the extracted instance,
    # and on config 2's m = 50 state the mode list and the bit pattern agree exactly
    st3 = W.full_state(3)
    sel = W.click_set(3, 0)
    p = T.probability(st3, sel, precision="128")
    want = T.torontonian(W.instance(3, 0, st3), "128")["value"] * math.sqrt(T.det_i_minus_a(st3))
    assert p == pytest.approx(want, rel=1e-12)
    st2 = W.full_state(2)
    sel2 = W.click_set(2)
    assert T.probability(st2, sel2, precision="128") == T.probability(st2, W.pattern_bits(sel2), precision="128")
    with pytest.raises(T.InvalidArgument):
        T.probability(st3, [3, 200], precision="128")  # mode outside the state


@pytest.mark.parametrize("prec", ["128", "256", "fp64"])
def test_device_list_folds_bit_identical(prec):
    # tor_torontonian with a device list (the reference's `workers`): the 64 top-level prefix
    # classes split across every listed device, one host thread per device, per-class partials
    # folded along the fixed tree -- bit-identical to one device.
    # (On a one-GPU box the list repeats device 0: the shards run concurrently there.)
    m = W.load_config_instance(2)
    one = T.torontonian(m, prec)
    for devs in ([0, 0], [0, 0, 0, 0], [0, 0, 0]):
        r = T.torontonian(m, prec, devices=devs)
        assert r["words"] == one["words"], devs
        assert r["sum_abs_terms"] == one["sum_abs_terms"]
        assert r["devices"] == len(devs)


@pytest.mark.gpu
def test_device_list_breakdown_reports_smallest_mask():
    # Breakdowns in several shards: the call reports the same (smallest) failing subset as one
    # device -- shard r covers prefix class r, and the first failing shard in class order wins.
    n = 24
    a = [0.1] * n
    c = [0.05] * n
    for j in (1, 2, 20, 21):  # four indefinite modes spread over the prefix classes
        a[j], c[j] = 0.5, 0.7
    m = diag_instance(n, a, c)
    with pytest.raises(T.BreakdownError) as one:
        T.torontonian(m, "128")
    for devs in ([0, 0], [0, 0, 0, 0], [0] * 8):
        with pytest.raises(T.BreakdownError) as e:
            T.torontonian(m, "128", devices=devs)
        assert (e.value.subset_mask, e.value.pivot_row) == (one.value.subset_mask, one.value.pivot_row), devs


@pytest.mark.parametrize("n", [9, 10, 12])
def test_tiny_positive_last_pivot_is_not_a_breakdown(n):
    """Tiny positive last-mode pivots (1 - a = 2^-44: det 2^-88) are eliminated, not reported
    as breakdowns.  The leaf's first-pivot test takes the sign of the word sum of the
    unnormalised state entry (round-1 advisor: the biased-grid DD leading word is a multiple
    of 2^-49, lazy QD leading words may cancel).  Diagonal A00 (closed form prod a/(1-a),
    test_torontonian.cpp:72-77).  DD's grid states carry ~2^-100 absolute error, so a 2x2
    block with det below that is indistinguishable from a breakdown in DD (as in fixed-128)."""
    a = [0.1] * (n - 1) + [1.0 - 2.0 ** -44]
    m = diag_instance(n, a)
    want = (1.0 / 9.0) ** (n - 1) * (2.0 ** 44 - 1.0)
    for prec in ("128", "256"):
        r = T.torontonian(m, prec)
        assert r["value"] == pytest.approx(want, rel=1e-9), prec
