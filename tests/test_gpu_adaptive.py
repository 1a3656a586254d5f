"""GPU tests of the adaptive-precision driver (AUTO) and of the FixedValue limbs at the C ABI.

select_precision (precision.cpp:80-121) sizes the width a priori; its lower-bound model is
blind on pure states (a_repr = 0 => b_lower = 0, precision.cpp:60), so AUTO adds a posterior
check: at least b_sgn bits must survive the cancellation sum|t| / |Tor| (after a log2(n) + 4
bit growth allowance), else DD re-runs in QD (escalated) and a QD result that still fails
raises PrecisionError "precision/insufficient".  Pure-state-like diagonal instances
(A00 = 0, A01 = c I) have the closed form Tor = prod_j (1/sqrt(1 - c^2) - 1) ~ (c^2/2)^n while
sum|t| = prod_j (1/sqrt(1 - c^2) + 1) ~ 2^n, so c sets the cancellation exactly.
"""
from __future__ import annotations

from decimal import Decimal, getcontext

import numpy as np
import pytest

import paper_2009_01177_b200 as T
from paper_2009_01177_b200 import workloads as W
from paper_2009_01177_b200.matrix import InputMatrix, _upper
from tests._util import fixed_value, within, words_value

pytestmark = pytest.mark.gpu
getcontext().prec = 120


def pure_diag(n, c):
    a00 = np.zeros((n, n), complex)
    a01 = np.diag(np.full(n, c, dtype=complex))
    return InputMatrix(n, _upper(a00), _upper(a01))


def closed_form(n, c):
    c = Decimal(float(c))  # the exact double the instance holds
    one = Decimal(1)
    f = one / (one - c * c).sqrt() - one
    return f ** n


def rel_err(words, want: Decimal) -> float:
    got = sum((Decimal(float(w)) for w in words), Decimal(0))
    return float(abs(got - want) / abs(want))


def test_auto_escalates_dd_to_qd_on_pure_state_cancellation():
    """n = 5, c = 1e-3: select_precision picks 128 (b_lower = 0), the sum cancels ~109 bits
    (more than DD's 104): AUTO must re-run in QD and return the QD value."""
    m = pure_diag(5, 1e-3)
    sel = T.select_precision(m)
    assert sel["width_bits"] == 128 and sel["b_lower"] == 0
    r = T.torontonian(m, "auto")
    assert r["escalated"] and r["mode"] == "qd" and r["width_bits"] == 256
    assert r["cancellation_bits"] == pytest.approx(109.4, abs=0.5)
    assert r["bits_left"] >= sel["b_sgn"]
    assert rel_err(r["words"], closed_form(5, 1e-3)) < 1e-25
    # forced DD reports the lost bits instead of escalating
    d = T.torontonian(m, "128")
    assert not d["escalated"] and d["bits_left"] < sel["b_sgn"]


def test_auto_escalation_matches_reference_fixed256():
    """The escalated value against the reference's own fixed-256 engine (oracle/_ref)."""
    ref = pytest.importorskip("oracle.ref")
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    m = pure_diag(5, 1e-3)
    g = ref.torontonian(m, "256")
    want = fixed_value(ref.limbs_to_int(g["raw_limbs"], 256), g["config"]["frac_bits"])
    r = T.torontonian(m, "auto")
    ok, rel = within(words_value(r["words"]), want, r["sum_abs_terms"], "qd")
    # fixed-256 keeps f ~ 250 fraction bits: 2^-180 sum|t| is far above its own error
    assert ok, f"err {rel:.3g} sum|t|"


def test_auto_raises_when_qd_is_exhausted():
    """n = 5, c = 1e-7: ~242 bits of cancellation exceed QD's 208."""
    m = pure_diag(5, 1e-7)
    with pytest.raises(T.PrecisionError) as e:
        T.torontonian(m, "auto")
    assert e.value.code == "precision/insufficient"
    q = T.torontonian(m, "256")  # an explicit width is returned as computed
    assert q["bits_left"] < 10


def test_exact_zero_dd_sum_escalates():
    """n = 4, c = 1e-4: Tor ~ 2^-110 ~ 2^-114 sum|t| -- the DD sum may cancel to exactly 0.0,
    which must count as no bits left (round 1 exempted value == 0.0); QD recovers it."""
    m = pure_diag(4, 1e-4)
    r = T.torontonian(m, "auto")
    assert r["escalated"] and r["mode"] == "qd"
    assert r["value"] != 0.0
    assert rel_err(r["words"], closed_form(4, 1e-4)) < 1e-20


def test_zero_input_is_exempt():
    """Tor(0) = 0 exactly (test_torontonian.cpp:49-61): no escalation, no error."""
    for n in (1, 5, 12):
        r = T.torontonian(pure_diag(n, 0.0), "auto")
        assert r["value"] == 0.0 and not r["escalated"] and r["mode"] == "dd"


def test_batch_auto_posterior_per_instance():
    """Batch AUTO applies the same check per instance: only the cancelling instance
    escalates; a QD-exhausted instance raises naming its index."""
    items = [W.generate_instance(5, 0.16, 0.06, 1), pure_diag(5, 1e-3), W.generate_instance(5, 0.16, 0.06, 2)]
    rs = T.torontonian_batch(items, "auto")
    assert [r["escalated"] for r in rs] == [False, True, False]
    assert [r["mode"] for r in rs] == ["dd", "qd", "dd"]
    for m, r in zip(items, rs):
        single = T.torontonian(m, "auto")
        assert r["words"] == single["words"]
    with pytest.raises(T.PrecisionError) as e:
        T.torontonian_batch(items + [pure_diag(5, 1e-7)], "auto")
    assert e.value.code == "precision/insufficient" and "instance 3" in str(e.value)


def test_batch_rejects_non_batch_modes():
    items = [W.generate_instance(5, 0.16, 0.06, 1)] * 2
    import ctypes as C
    ins = [T.api._In(m) for m in items]
    arr = (T.api.TorInput * 2)(*[i.s for i in ins])
    res = (T.api.TorResult * 2)()
    for bad in (4, 5, 9, -3):
        err = T.api.TorError()
        st = T.api.lib().tor_torontonian_batch(arr, 2, bad, 0, res, C.byref(err))
        assert st == 1 and err.code.decode() == "precision/range"


# ------------------------------------------------------------------- raw limbs --
@pytest.mark.parametrize("name", ["gen10_s1", "gen12_s7", "cfg1", "cfg2"])
def test_raw_limbs_in_float_modes(name, golden):
    """tor_result.raw_limbs in DD/QD: the words re-quantised exactly at config.frac_bits
    (torontonian.hpp:14-29 FixedValue), within the mode's tolerance of the reference's own
    accumulator limbs."""
    from tests.test_gpu_parity import small_instance
    g = golden[name]
    m = small_instance(name)
    for prec, key, mode in (("128", "fixed128", "dd"), ("256", "fixed256", "qd")):
        r = T.torontonian(m, prec)
        wb, f = r["width_bits"], r["config"]["frac_bits"]
        assert r["raw_limbs"] == T.api.raw_limbs(r["words"], wb, f)  # C == exact Python
        raw = 0
        for i in reversed(range(wb // 64)):
            raw = (raw << 64) | r["raw_limbs"][i]
        if raw >> (wb - 1):
            raw -= 1 << wb
        ok, rel = within(fixed_value(raw, f), fixed_value(g[key]["raw"], g[key]["frac_bits"]),
                         r["sum_abs_terms"], mode)
        assert ok, f"{name} {mode}: {rel:.3g}"
    assert T.torontonian(m, "fp64")["raw_limbs"] == (0, 0, 0, 0)


def test_raw_limbs_negative_values():
    """Two's complement for a negative Torontonian: A00 = diag(-0.1, -0.2, -0.3) gives
    Tor = prod a/(1-a) < 0 (test_torontonian.cpp:72-77's closed form with negated a)."""
    a = [-0.1, -0.2, -0.3]
    m = InputMatrix(3, _upper(np.diag(np.array(a, complex))), _upper(np.zeros((3, 3), complex)))
    want = float(np.prod([x / (1 - x) for x in a]))
    for prec in ("128", "256"):
        r = T.torontonian(m, prec)
        assert r["value"] == pytest.approx(want, rel=1e-14) and r["value"] < 0
        assert r["raw_limbs"] == T.api.raw_limbs(r["words"], r["width_bits"], r["config"]["frac_bits"])
        wb = r["width_bits"]
        assert r["raw_limbs"][wb // 64 - 1] >> 63 == 1  # sign bit of the top limb
    # (no fixed-point comparison: det(I - A) > 1 here, so force_width's f = width - 1 - b_upper
    # leaves no integer bit and the reference's own fixed-point path overflows)
