"""CPU: pin the oracle restatement (oracle/tor_oracle.c) to the reference's golden values.

The oracle is the checker for the GPU parity tests; it must reproduce the unmodified
reference (tests/golden/reference_values.json, written through oracle/_ref) limb-exact.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import port
from paper_2009_01177_b200 import workloads as W
from paper_2009_01177_b200.matrix import InputMatrix, _upper
from tests.test_gpu_parity import GEN_CASES, diag_instance, small_instance

FAST = [c for c in GEN_CASES if c not in ("cfg2",)]


@pytest.mark.parametrize("name", FAST)
def test_fixed_point_engine_limb_exact(name, golden):
    g = golden[name]
    m = small_instance(name)
    for p in ("128", "256"):
        r = port.torontonian(m, p)
        assert r["raw"] == int(g[f"fixed{p}"]["raw"]), f"{name} fixed-{p}"
        assert r["config"]["frac_bits"] == g[f"fixed{p}"]["frac_bits"]


@pytest.mark.parametrize("name", FAST)
def test_fp64_oracle_bit_exact(name, golden):
    m = small_instance(name)
    assert port.torontonian_reference(m) == golden[name]["fp64_reference"]


@pytest.mark.parametrize("name", FAST + ["cfg2"])
def test_precision_selection_identical(name, golden):
    g = golden[name]
    m = small_instance(name)
    sel = port.select_precision(m)
    for k, v in g["select_precision"].items():
        if k != "alpha":
            assert sel[k] == v, k
    for w in (128, 256):
        want = g[f"force_width_{w}"]
        got = port.force_width(m, w)
        for k, v in want.items():
            if k != "alpha":
                assert got[k] == v, (w, k)


@pytest.mark.parametrize("n", range(1, 11))
def test_zero_matrix(n, golden):
    m = diag_instance(n, [0.0] * n)
    r = port.torontonian(m, "auto")
    assert r["raw"] == 0 and r["value"] == 0.0
    assert int(golden[f"zero_{n}"]["fixedauto"]["raw"]) == 0
    assert port.torontonian_reference(m) == 0.0


def test_closed_forms():
    """test_torontonian.cpp:63-81."""
    assert port.torontonian(diag_instance(1, [0.5]))["value"] == pytest.approx(1.0, rel=1e-12)
    one = port.torontonian(diag_instance(1, [0.3], [0.1]))["value"]
    assert one == pytest.approx(1.0 / math.sqrt(0.7 * 0.7 - 0.01) - 1.0, rel=1e-12)
    three = port.torontonian(diag_instance(3, [0.1, 0.2, 0.3]))["value"]
    assert three == pytest.approx((0.1 / 0.9) * (0.2 / 0.8) * (0.3 / 0.7), rel=1e-12)


def test_breakdown_matches_reference(golden):
    """Forced 128-bit on the near-singular stress instance breaks down in fixed point
    (test_torontonian.cpp:218-244); 256 bits succeeds with the reference's value."""
    g = golden["breakdown6"]
    m = small_instance("breakdown6")
    with pytest.raises(port.OracleError) as e:
        port.torontonian(m, "128", threads=1)
    assert e.value.code == "linalg/breakdown" == g["fixed128"]["error"]
    r = port.torontonian(m, "256")
    assert r["raw"] == int(g["fixed256"]["raw"])


def test_cfg3_items(golden):
    for i, g in list(sorted(golden["cfg3_items"].items(), key=lambda kv: int(kv[0])))[:4]:
        m = W.load_config_instance(3, int(i))
        assert port.torontonian(m, "128")["raw"] == int(g["fixed128"]["raw"])
        assert port.torontonian_reference(m) == g["fp64_reference"]


@pytest.mark.parametrize("cfg", ["cfg4_slices", "cfg5_slices"])
def test_large_n_slices_limb_exact(cfg, golden):
    g = golden[cfg]
    m = W.load_config_instance(4 if cfg == "cfg4_slices" else 5)
    gw = g["widths"]["128"]
    for c in gw["classes"][:2]:
        tot, per, sabs = port.slice(m, 128, gw["frac_bits"], g["k"], c["cls"], c["cls"] + 1)
        assert per[0] == int(c["raw"])
        assert sabs[0] == pytest.approx(c["sum_abs"], rel=1e-12)


def test_subsets():
    """test_subsets.cpp / tests/python/test_smoke.py subset pins."""
    assert port.binom(50, 25) == 126410606437752
    assert port.get_next_mask(0b010011) == 0b001110
    mask = port.get_kth_mask(8, 3, 0)
    seen = 0
    while mask:
        seen += 1
        mask = port.get_next_mask(mask)
    assert seen == math.comb(8, 3)


def test_fixed_point_primitives_vs_big_integers():
    """test_fixed_point.cpp:130-200 analogue: mul = floor(ab/2^f) mod 2^w, rsqrt bracket."""
    rng = np.random.default_rng(7)
    for width in (128, 256):
        f = width - 20
        for _ in range(300):
            a = int(rng.integers(0, 1 << 62)) << int(rng.integers(0, width - 70))
            b = int(rng.integers(0, 1 << 62)) << int(rng.integers(0, width - 70))
            a = -a if rng.random() < 0.5 else a
            b = -b if rng.random() < 0.5 else b
            want = (a * b) >> f
            want = ((want + (1 << (width - 1))) % (1 << width)) - (1 << (width - 1))
            assert port.wide_mul(a, b, width, f) == want
        for _ in range(50):
            a = int(rng.integers(1, 1 << 30)) << (f - 20)
            r = port.wide_rsqrt(a, width, f)
            target = 1 << (3 * f)
            assert (r - 2) ** 2 * a <= target <= (r + 2) ** 2 * a
