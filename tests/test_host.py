"""CPU: the C-ABI library, the host-side port of the reference logic, the data model.

No compute calls need a GPU here: the library must load and export every symbol
include/tor_capi.h declares; validation / precision selection / symmetry checks /
folds are host code and must equal the reference bit-for-bit; the evaluation entry
points must FAIL LOUDLY without a device (no CPU fallback).
"""
from __future__ import annotations

import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_2009_01177_b200 as T
from paper_2009_01177_b200 import api, subsets
from paper_2009_01177_b200 import workloads as W
from paper_2009_01177_b200.matrix import load_matrix_bytes, save_matrix
from tests.test_gpu_parity import GEN_CASES, diag_instance, small_instance

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "tor_capi.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|uint64_t)\s+(tor_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(api.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 17
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(api.EXPORTS)
    assert lib.tor_abi_version() == 1


def test_library_is_sm100a_native():
    """The shipped library carries sm_100a SASS for the engine kernels."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", api.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", GEN_CASES)
def test_precision_port_identical_to_reference(name, golden):
    g = golden[name]
    m = small_instance(name)
    sel = T.select_precision(m)
    for k, v in g["select_precision"].items():
        if k != "alpha":
            assert sel[k] == v, k
    for w in (128, 256):
        got = T.force_width(m, w)
        for k, v in g[f"force_width_{w}"].items():
            if k != "alpha":
                assert got[k] == v, (w, k)
    assert T.det_i_minus_a(m) == g["det_i_minus_a"]


@pytest.mark.parametrize("cfg", ["cfg4", "cfg5"])
def test_precision_port_large_configs(cfg, golden):
    g = golden[cfg]
    m = W.load_config_instance(int(cfg[-1]))
    sel = T.select_precision(m)
    for k, v in g["select_precision"].items():
        if k != "alpha":
            assert sel[k] == v, k
    assert T.det_i_minus_a(m) == g["det_i_minus_a"]


def test_precision_pins():
    """test_precision.cpp pins (26-154)."""
    assert T.select_precision(T.generate_instance(4, 0.16, 0.06, 2026))["b_accum"] == 7
    c = T.select_precision(T.generate_instance(4, 0.16, 0.06, 2026), sig_decimal_digits=6)
    assert c["b_sgn"] == 20
    assert T.select_precision(T.generate_instance(30, 0.05, 0.02, 11))["width_bits"] == 256
    assert T.select_precision(T.generate_instance(45, 0.16, 0.06, 3))["width_bits"] == 256
    with pytest.raises(T.PrecisionError) as e:
        T.select_precision(T.generate_instance(55, 0.01, 0.004, 5))
    assert e.value.code == "precision/unsupported"
    half = diag_instance(2, [0.5, 0.5])
    assert T.force_width(half, 128)["frac_bits"] == 123
    assert T.force_width(half, 256)["frac_bits"] == 251
    with pytest.raises(T.InvalidArgument):
        T.force_width(half, 192)
    with pytest.raises(T.PrecisionError) as e:
        T.force_width(diag_instance(10, [0.999] * 10), 128)
    assert e.value.code == "precision/scaling"


def test_generator_matches_reference_inputs(golden):
    """Our restated xoshiro256** generator reproduces the reference instances: the
    reference's own values for them are reproduced limb-exact by the oracle."""
    from oracle import port
    for name, seed in (("gen10_s1", 1), ("gen10_s2", 2), ("gen8_s99", 99)):
        n = 8 if seed == 99 else 10
        m = T.generate_instance(n, 0.16, 0.06, seed)
        assert port.torontonian(m, "128")["raw"] == int(golden[name]["fixed128"]["raw"])


def test_evaluation_fails_loudly_without_gpu():
    if T.device_count() > 0:
        pytest.skip("GPU present")
    m = W.load_config_instance(1)
    with pytest.raises(T.DeviceError):
        T.torontonian(m, "128")
    with pytest.raises(T.DeviceError):
        T.torontonian_reference(m)


def test_validation_errors_before_device():
    skew = diag_instance(2, [0.2, 0.2])
    skew.a00[0] = 0.2 + 0.05j
    with pytest.raises(T.TorfpError) as e:
        T.torontonian(skew)
    assert e.value.code == "torontonian/symmetry"
    with pytest.raises(T.InvalidArgument):
        T.torontonian(diag_instance(41, [0.0] * 41))
    with pytest.raises(T.InvalidArgument):
        T.torontonian_reference(diag_instance(21, [0.0] * 21))
    with pytest.raises(T.PrecisionError) as e:
        T.torontonian(diag_instance(1, [0.5], [0.7]))
    assert e.value.code == "precision/det-nonpositive"


def test_fold_partials_is_host_side_and_order_fixed():
    """tor_fold_partials runs on the host: folding 2^k shard partials of exactly
    representable values gives their exact sum regardless of grouping."""
    m = W.load_config_instance(1)
    vals = [1.0, -0.5, 0.25, 2.0 ** -60, -(2.0 ** -61), 3.0, -3.0, 2.0 ** -100]
    parts = [dict(mode=api.PREC_DD, class_bits=3, class_lo=i, class_hi=i + 1, words=(v, 0.0, 0.0, 0.0),
                  sum_abs=abs(v), term_count=1 << 13) for i, v in enumerate(vals)]
    r = T.fold_partials(parts, m)
    assert api.words_fraction(r["words"]) == sum(api.words_fraction((v,)) for v in vals)
    assert r["term_count"] == 1 << 16


def test_raw_limbs_requantisation():
    assert api.raw_limbs((0.5, 0.0), 128, 10) == (512, 0, 0, 0)
    assert api.raw_limbs((-1.0, 0.0), 128, 4) == ((1 << 64) - 16, (1 << 64) - 1, 0, 0)


# ------------------------------------------------------------ data model ----
def test_from_dense_and_symmetry_gate():
    m = T.generate_instance(5, 0.2, 0.05, 11)
    d = m.to_dense()
    back = T.from_dense(d)
    assert np.array_equal(back.a00, m.a00) and np.array_equal(back.a01, m.a01)
    bad = np.zeros((4, 4), complex)
    bad[0, 1] = 0.1
    with pytest.raises(T.TorfpError):
        T.from_dense(bad)
    assert T.check_symmetries(m)["pass"]


def test_gbsa_text_roundtrip_lossless():
    m = W.load_config_instance(4)
    back = load_matrix_bytes(save_matrix(m, "text"))
    assert np.array_equal(back.a00, m.a00) and np.array_equal(back.a01, m.a01)


def test_gbsa_binary_quantised(tmp_path):
    """tests/python/test_smoke.py:83-93."""
    m = T.generate_instance(5, 0.2, 0.05, 11)
    p = str(tmp_path / "m.gbsa")
    m.save(p, format="binary", bits=32)
    back = T.load_matrix(p)
    assert back.n_modes == 5 and back.quant_bits == 32
    assert np.allclose(back.to_dense(), m.to_dense(), atol=2 ** -32)
    assert T.check_symmetries(back)["pass"]
    assert T.quantize(0.5, 16) == 16384 and T.dequantize(16384, 16) == 0.5
    with pytest.raises(T.TorfpError):
        T.quantize(1.0, 16)


def test_extract_submatrix():
    m = T.generate_instance(6, 0.16, 0.06, 5)
    sub = T.extract_submatrix(m, 0b000101)
    keep = [0, 2, 6, 8]
    assert np.allclose(sub.to_dense(), m.to_dense()[np.ix_(keep, keep)])


def test_subset_api():
    assert T.binom(50, 25) == 126410606437752
    assert T.get_next_mask(0b010011) == 0b001110
    counts = [[c for (_, _, c) in T.partition(12, r, 7)] for r in range(7)]
    for z in range(12):
        col = [counts[r][z] for r in range(7)]
        assert sum(col) == math.comb(12, z + 1) and max(col) - min(col) <= 1
    assert T.total_op_count(1) == 12 and T.factorization_op_count(4) == 96
    assert subsets.prefix_classes(32, 3, 8) == (3, 3, 4)


def test_config_fixtures_reproduce_survey_values(golden):
    """The committed BASELINE inputs are the survey's recipe: reference values pinned."""
    assert golden["cfg1"]["fixed128"]["value"] == 6.5025695289866082e-05
    assert golden["cfg2"]["fixed128"]["value"] == 1.1801356334058375e-07
    assert golden["cfg3_items"]["0"]["fixed128"]["value"] == pytest.approx(1.2392775476016946e-10, rel=1e-15)


def test_batch_validation_errors_before_device():
    # the batch validates its instances on host threads; the first bad instance in index
    # order is reported, before any device work
    good = [diag_instance(3, [0.1, 0.2, 0.3]) for _ in range(300)]
    skew = diag_instance(3, [0.1, 0.2, 0.3])
    skew.a00[0] = 0.1 + 0.05j
    with pytest.raises(T.TorfpError) as e:
        T.torontonian_batch(good[:150] + [skew] + good[150:] + [diag_instance(4, [0.1] * 4)], "128")
    assert e.value.code == "torontonian/symmetry"
    with pytest.raises(T.InvalidArgument) as e:
        T.torontonian_batch(good + [diag_instance(4, [0.1] * 4)] + good[:10], "fp64")
    assert e.value.code == "torontonian/range"


def test_slice_range_beyond_reference_limit():
    # tor_torontonian keeps the reference's N <= 40; slices/shards/plans accept N <= 50
    with pytest.raises(T.InvalidArgument):
        T.torontonian(diag_instance(41, [0.1] * 41), "128")
    with pytest.raises(T.InvalidArgument) as e:
        T.torontonian_slice(diag_instance(51, [0.1] * 51), "128", 30, 0, 1)
    assert "50" in str(e.value)
    if T.device_count() == 0:
        with pytest.raises(T.DeviceError):  # validated, then needs the device
            T.torontonian_slice(diag_instance(50, [0.1] * 50), "128", 30, 0, 1)


@pytest.mark.parametrize("im", [0.0, 1e-13, 4.9e-13, 5e-13, 5.1e-13, 1e-12, 3e-12])
def test_symmetry_gate_without_dense_matrix_matches_dense(im):
    """The evaluation entry points gate inputs with check_symmetries_tri (O(n), no dense
    matrix); it must decide exactly as the dense check_symmetries (matrix_io.cpp:285-305) that
    tor_check_symmetries runs: only the A00 diagonal's imaginary parts can deviate."""
    m = W.generate_instance(6, 0.16, 0.06, 3)
    a00 = m.a00.copy()
    a00[T.matrix.tri_index(6, 2, 2)] += 1j * im
    bad = T.InputMatrix(6, a00, m.a01)
    dense = T.check_symmetries(bad)
    assert dense["hermitian_dev"] == pytest.approx(2 * im, rel=1e-15, abs=0)
    try:
        T.torontonian(bad, "128")
        gate_pass = True
    except T.DeviceError:
        gate_pass = True  # passed validation, no GPU here
    except T.TorfpError as e:
        assert e.code == "torontonian/symmetry"
        gate_pass = False
    assert gate_pass == dense["pass"]
