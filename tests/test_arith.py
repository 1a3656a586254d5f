"""Unit tests of the engine's multi-word arithmetic (csrc/arith.cuh) against exact rationals.

The same header the sm_100a kernels compile is built for the host (tests/harness/
arith_harness.cpp, g++ -ffp-contract=off; the MUFU seed is emulated at its ~2^-20 accuracy,
so the Newton steps run on the device code path) and every primitive is checked against
Fraction arithmetic: biased-grid DD rank-1/rank-2 Schur updates, DD products, reciprocal
square roots, 2x2 determinants, the pivot chain and leaf term, the lazy DD accumulator, and
the QD add / mul / rank-2 / rsqrt / pivot.  Error bounds are the ones the parity tolerances
rely on (DD ~2^-100, QD ~2^-200)."""
from __future__ import annotations

import ctypes as C
import math
import os
import random
import subprocess
from fractions import Fraction

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
D2 = C.c_double * 2
D4 = C.c_double * 4


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("arith") / "libarith_host.so")
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-shared", "-fPIC", "-o", out,
                    os.path.join(HERE, "harness", "arith_harness.cpp")], check=True)
    L = C.CDLL(out)
    L.h_grid_c.restype = C.c_double
    L.h_dd_to_grid.argtypes = [C.c_double, C.c_double, C.c_void_p]
    return L


def F(words) -> Fraction:
    return sum((Fraction(w) for w in words), Fraction(0))


def rsqrt_exact(x: Fraction, bits: int = 320) -> Fraction:
    # floor(2^bits / sqrt(x)) / 2^bits
    return Fraction(math.isqrt((1 << (2 * bits)) * x.denominator // x.numerator), 1 << bits)


def rand_dd(rng, lo, hi):
    h = rng.uniform(lo, hi)
    return [h, rng.uniform(-0.5, 0.5) * math.ulp(h)]


def rand_qd(rng, lo, hi):
    w = [rng.uniform(lo, hi)]
    for _ in range(3):
        w.append(rng.uniform(-0.5, 0.5) * math.ulp(w[-1]))
    return w


def test_grid_entry_roundtrip(lib):
    rng = random.Random(1)
    C0 = lib.h_grid_c()
    for _ in range(500):
        x, y = rng.uniform(-3.7, 3.7), rng.uniform(-1e-3, 1e-3)
        o = D2()
        lib.h_dd_to_grid(x, y, o)
        assert 8.0 <= o[0] < 16.0 and (Fraction(o[0]) * 2 ** 49).denominator == 1  # biased, on the grid
        assert F([o[0] - C0, o[1]]) == Fraction(x) + Fraction(y)  # exact


def test_dd_rank2_and_rank1_grid(lib):
    rng = random.Random(2)
    C0 = Fraction(lib.h_grid_c())
    worst = 0.0
    for _ in range(2000):
        x = rng.uniform(-1.0, 1.0)
        s = D2()
        lib.h_dd_to_grid(x, rng.uniform(-1, 1) * 2.0 ** -52, s)
        a, b, c, d = (D2(*rand_dd(rng, -1.3, 1.3)) for _ in range(4))
        o = D2()
        lib.h_dd_rank2(s, a, b, c, d, o)
        assert 8.0 <= o[0] < 16.0 and (Fraction(o[0]) * 2 ** 49).denominator == 1
        exact = F(s) - C0 - F(a) * F(b) - F(c) * F(d)
        err = abs(F(o) - C0 - exact)
        worst = max(worst, float(err))
        o1 = D2()
        lib.h_dd_rank1s(s, a, b, o1)  # unbiased result
        assert abs(F(o1) - (F(s) - C0 - F(a) * F(b))) <= 2.0 ** -100
    assert worst <= 2.0 ** -100, worst


def test_dd_mul_rsqrt_det(lib):
    rng = random.Random(3)
    for _ in range(2000):
        a, b = D2(*rand_dd(rng, -2, 2)), D2(*rand_dd(rng, -2, 2))
        o = D2()
        lib.h_dd_mul(a, b, o)
        ex = F(a) * F(b)
        assert abs(F(o) - ex) <= 2.0 ** -103 * abs(ex)
        x = D2(*rand_dd(rng, 2.0 ** -30, 4.0))
        lib.h_dd_rsqrt(x, o)
        r = rsqrt_exact(F(x))
        assert abs(F(o) - r) <= 2.0 ** -102 * r
        # det of an SPD 2x2 [[p, q], [q, s]]
        p = rng.uniform(0.1, 3.0)
        s_ = rng.uniform(0.1, 3.0)
        q = rng.uniform(-1, 1) * math.sqrt(p * s_) * 0.999
        A, B, S = (D2(v, rng.uniform(-0.5, 0.5) * math.ulp(v)) for v in (p, q, s_))
        lib.h_dd_det2(A, B, S, o)
        ex = F(A) * F(S) - F(B) * F(B)
        assert abs(F(o) - ex) <= 2.0 ** -102 * (F(A) * F(S) + F(B) * F(B))
        assert o[0] == o[0] + o[1]  # normalised


def _spd2_biased(lib, rng):
    p = rng.uniform(0.05, 3.5)
    s_ = rng.uniform(0.05, 3.5)
    q = rng.uniform(-1, 1) * math.sqrt(p * s_) * 0.99
    out = []
    for v in (p, q, s_):
        e = D2()
        lib.h_dd_to_grid(v, rng.uniform(-1, 1) * 2.0 ** -60, e)
        out.append(e)
    return out


def test_dd_pivot_and_leaf(lib):
    rng = random.Random(4)
    C0 = Fraction(lib.h_grid_c())
    for _ in range(1000):
        s00, s01, s11 = _spd2_biased(lib, rng)
        t = D2(*rand_dd(rng, 1e-3, 10.0))
        o = (C.c_double * 8)()
        assert lib.h_dd_pivot(s00, s01, s11, t, o) == 0
        a, b, c = F(s00) - C0, F(s01) - C0, F(s11) - C0
        det = a * c - b * b
        # state entries carry absolute precision (~2^-100 of the O(1) scale): results are
        # bounded relative to the scale, amplified by the 2x2 condition (a c + b^2) / det
        # (the low*low products of un-normalised grid words, <= 2^-100 absolute, are dropped
        # from det: a further 2^-100 / det relative)
        kap = float((a * c + b * b) / det) + float(1 / det)
        r1, rd = rsqrt_exact(a), rsqrt_exact(det)
        assert abs(F(o[0:2]) - r1) <= 2.0 ** -100 * r1 * (1 + float(1 / a))
        assert abs(F(o[2:4]) - b * r1) <= 2.0 ** -99 * r1
        r2 = rsqrt_exact(c - b * b / a)
        assert abs(F(o[4:6]) - r2) <= 2.0 ** -97 * r2 * kap
        tn = F(t) * rd
        assert abs(F(o[6:8]) - tn) <= 2.0 ** -97 * tn * kap
        lf = D2()
        assert lib.h_dd_leaf(s00, s01, s11, t, lf) == 0
        assert abs(F(lf) - tn) <= 2.0 ** -97 * tn * kap


def test_dd_pivot_flags_nonpositive(lib):
    e = [D2() for _ in range(3)]
    lib.h_dd_to_grid(1.0, 0.0, e[0])
    lib.h_dd_to_grid(1.0, 0.0, e[1])
    lib.h_dd_to_grid(0.5, 0.0, e[2])  # det = 0.5 - 1 < 0
    o = (C.c_double * 8)()
    assert lib.h_dd_pivot(e[0], e[1], e[2], D2(1.0, 0.0), o) == 2
    lib.h_dd_to_grid(-1.0, 0.0, e[0])
    assert lib.h_dd_pivot(e[0], e[1], e[2], D2(1.0, 0.0), o) & 1


def test_dd_accumulator(lib):
    rng = random.Random(5)
    n = 4096
    terms = [rand_dd(rng, 1e-6, 1.0) for _ in range(n)]
    negs = [rng.random() < 0.5 for _ in range(n)]
    buf = (C.c_double * (2 * n))(*[w for t in terms for w in t])
    ng = (C.c_int * n)(*negs)
    o = (C.c_double * 3)()
    lib.h_dd_acc(buf, ng, n, 16, o)
    exact = sum(((-F(t)) if s else F(t) for t, s in zip(terms, negs)), Fraction(0))
    sabs = sum(abs(t[0]) for t in terms)
    assert abs(F(o[0:2]) - exact) <= 2.0 ** -98 * sabs
    assert o[2] == pytest.approx(sabs, rel=1e-12)


def test_qd_ops(lib):
    rng = random.Random(6)
    for _ in range(1000):
        a, b = D4(*rand_qd(rng, -2, 2)), D4(*rand_qd(rng, -2, 2))
        o = D4()
        lib.h_qd_add(a, b, o)
        ex = F(a) + F(b)
        assert abs(F(o) - ex) <= 2.0 ** -200 * (abs(F(a)) + abs(F(b)))
        lib.h_qd_mul(a, b, o)
        ex = F(a) * F(b)
        assert abs(F(o) - ex) <= 2.0 ** -200 * abs(ex)
        lib.h_qd_mul_fused(a, b, o)  # the engine's product (Arith<qd>::mul)
        assert abs(F(o) - ex) <= 2.0 ** -204 * abs(ex)
        s, c, d = (D4(*rand_qd(rng, -1.5, 1.5)) for _ in range(3))
        lib.h_qd_rank2(s, a, b, c, d, o)
        ex = F(s) - F(a) * F(b) - F(c) * F(d)
        assert abs(F(o) - ex) <= 2.0 ** -204 * (abs(F(s)) + abs(F(a) * F(b)) + abs(F(c) * F(d)))
        x = D4(*rand_qd(rng, 2.0 ** -20, 4.0))
        lib.h_qd_rsqrt(x, o)
        r = rsqrt_exact(F(x))
        assert abs(F(o) - r) <= 2.0 ** -204 * r


def test_qd_pivot(lib):
    rng = random.Random(7)
    for _ in range(300):
        p = rng.uniform(0.05, 3.5)
        s_ = rng.uniform(0.05, 3.5)
        q = rng.uniform(-1, 1) * math.sqrt(p * s_) * 0.99
        s00, s01, s11 = (D4(*rand_qd(rng, v, v)) for v in (p, q, s_))
        t = D4(*rand_qd(rng, 1e-3, 10.0))
        o = (C.c_double * 16)()
        assert lib.h_qd_pivot(s00, s01, s11, t, o) == 0
        a, b, c = F(s00), F(s01), F(s11)
        det = a * c - b * b
        kappa = 1 + float(a * c / det)
        assert abs(F(o[0:4]) - rsqrt_exact(a)) <= 2.0 ** -198 * rsqrt_exact(a)
        tn = F(t) * rsqrt_exact(det)
        assert abs(F(o[12:16]) - tn) <= 2.0 ** -196 * tn * kappa


def test_qd_lazy_state_chain(lib):
    # Schur-state entries are updated up to n times without renormalisation (words ordered
    # by absolute scale); the absolute error stays at the ~2^-200 level of the O(1) scale
    rng = random.Random(8)
    for _ in range(50):
        s = D4(*rand_qd(rng, -1.0, 1.0))
        exact = F(s)
        for _ in range(40):
            a, b, c, d = (D4(*rand_qd(rng, -0.3, 0.3)) for _ in range(4))
            o = D4()
            lib.h_qd_rank2(s, a, b, c, d, o)
            exact -= F(a) * F(b) + F(c) * F(d)
            s = o
        assert abs(F(s) - exact) <= 2.0 ** -200


def test_qd_accumulator(lib):
    rng = random.Random(9)
    n = 4096
    terms = [rand_qd(rng, 1e-6, 1.0) for _ in range(n)]
    negs = [rng.random() < 0.5 for _ in range(n)]
    buf = (C.c_double * (4 * n))(*[w for t in terms for w in t])
    ng = (C.c_int * n)(*negs)
    o = (C.c_double * 5)()
    lib.h_qd_acc(buf, ng, n, 8, o)
    exact = sum(((-F(t)) if s else F(t) for t, s in zip(terms, negs)), Fraction(0))
    sabs = sum(abs(t[0]) for t in terms)
    assert abs(F(o[0:4]) - exact) <= 2.0 ** -200 * sabs


def test_qd_products_of_cancelled_lazy_entries(lib):
    # a lazy (unrenormalised) state entry whose leading word has cancelled -- words ordered by
    # absolute scale, the second word larger than the first -- times normalised factors:
    # the pivot-row vector pair stays exact to the ~2^-200 absolute level
    rng = random.Random(10)
    for _ in range(300):
        small = rng.uniform(-1, 1) * 2.0 ** rng.randint(-70, -45)
        s0 = D4(small, rng.uniform(-1, 1) * 2.0 ** -50, rng.uniform(-1, 1) * 2.0 ** -103,
                rng.uniform(-1, 1) * 2.0 ** -156)
        s1 = D4(*rand_qd(rng, -1.0, 1.0))
        r1, u1, r2 = (D4(*rand_qd(rng, 0.5, 2.0)) for _ in range(3))
        u, w = D4(), D4()
        lib.h_qd_vec(s0, s1, r1, u1, r2, u, w)
        eu = F(s0) * F(r1)
        ew = (F(s1) - F(u1) * eu) * F(r2)
        assert abs(F(u) - eu) <= 2.0 ** -200
        assert abs(F(w) - ew) <= 2.0 ** -198
