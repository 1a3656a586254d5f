"""TEST INFRASTRUCTURE ONLY: ctypes bindings to oracle/_ref/libtorfp_ref.so.

libtorfp_ref.so is the UNMODIFIED reference engine (torfp) compiled from
/root/reference/proj/src by oracle/Makefile, plus our C harness
(oracle/ref_harness.cpp).  Only tests/, bench.py's reference / cpu_baseline
legs and tests/golden/make_golden.py may import this module; the product
library never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libtorfp_ref.so")

_lib = None


class RefError(RuntimeError):
    def __init__(self, status, code, msg, mask=0, row=-1):
        super().__init__(f"[{status}] {code}: {msg}")
        self.status, self.code, self.msg, self.mask, self.row = status, code, msg, mask, row


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref)")
        _lib = C.CDLL(LIB_PATH)
    return _lib


def _err():
    return (C.create_string_buffer(64), C.create_string_buffer(256), C.c_uint64(0), C.c_int64(-1))


def _call(fn, *args):
    code, msg, mask, row = _err()
    st = fn(*args, code, 64, msg, 256, C.byref(mask), C.byref(row))
    if st != 0:
        raise RefError(st, code.value.decode(), msg.value.decode(), mask.value, row.value)


def _tri(m):
    a00, a01 = m.interleaved()
    return (a00.ctypes.data_as(C.POINTER(C.c_double)), a01.ctypes.data_as(C.POINTER(C.c_double)),
            (a00, a01))


def _cfg(ints, dbls):
    return dict(width_bits=ints[0], frac_bits=ints[1], b_lower=ints[2], b_upper=ints[3],
                b_sgn=ints[4], b_accum=ints[5], a_repr=dbls[0], k_corr=dbls[1], alpha=dbls[2])


def torontonian(m, precision="auto", workers=0):
    """Reference torontonian() (torontonian.cpp:151) -> dict like bindings.cpp:69-85."""
    p = {"auto": 0, "128": 1, "256": 2}[str(precision)]
    a00, a01, keep = _tri(m)
    val = C.c_double()
    limbs = (C.c_uint64 * 4)()
    wb = C.c_int()
    ints = (C.c_int * 6)()
    dbls = (C.c_double * 3)()
    ctr = (C.c_uint64 * 4)()
    tc = C.c_uint64()
    wall = C.c_double()
    wo = C.c_int()
    _call(lib().ref_torontonian, C.c_int(m.n_modes), a00, a01, C.c_int(p), C.c_int(workers),
          C.byref(val), limbs, C.byref(wb), ints, dbls, ctr, C.byref(tc), C.byref(wall), C.byref(wo))
    return dict(value=val.value, raw_limbs=tuple(int(x) for x in limbs), width_bits=wb.value,
                config=_cfg(ints, dbls), term_count=tc.value,
                counters=dict(mults=ctr[0], adds=ctr[1], recips=ctr[2], rsqrts=ctr[3]),
                wall_seconds=wall.value, workers=wo.value)


def torontonian_reference(m):
    a00, a01, keep = _tri(m)
    v = C.c_double()
    _call(lib().ref_torontonian_reference, C.c_int(m.n_modes), a00, a01, C.byref(v))
    return v.value


def reference_timed(m):
    a00, a01, keep = _tri(m)
    v = C.c_double()
    s = C.c_double()
    _call(lib().ref_reference_timed, C.c_int(m.n_modes), a00, a01, C.byref(v), C.byref(s))
    return v.value, s.value


def select_precision(m, N=None, sig=3, alpha=0.5):
    a00, a01, keep = _tri(m)
    ints = (C.c_int * 6)()
    dbls = (C.c_double * 3)()
    _call(lib().ref_select_precision, C.c_int(m.n_modes), a00, a01,
          C.c_int(m.n_modes if N is None else N), C.c_int(sig), C.c_double(alpha), ints, dbls)
    return _cfg(ints, dbls)


def force_width(m, width):
    a00, a01, keep = _tri(m)
    ints = (C.c_int * 6)()
    dbls = (C.c_double * 3)()
    _call(lib().ref_force_width, C.c_int(m.n_modes), a00, a01, C.c_int(width), ints, dbls)
    return _cfg(ints, dbls)


def det_i_minus_a_float(m):
    a00, a01, keep = _tri(m)
    v = C.c_double()
    _call(lib().ref_det_i_minus_a_float, C.c_int(m.n_modes), a00, a01, C.byref(v))
    return v.value


def check_symmetries(m):
    a00, a01, keep = _tri(m)
    devs = (C.c_double * 3)()
    ok = C.c_int()
    _call(lib().ref_check_symmetries, C.c_int(m.n_modes), a00, a01, devs, C.byref(ok))
    return dict(hermitian_dev=devs[0], a01_sym_dev=devs[1], block_conj_dev=devs[2],
                tolerance=1e-12, **{"pass": bool(ok.value)})


def generate_instance(n, a_target, spread, seed):
    from paper_2009_01177_b200.matrix import InputMatrix
    t = n * (n + 1) // 2
    a00 = np.zeros(2 * t)
    a01 = np.zeros(2 * t)
    _call(lib().ref_generate_instance, C.c_int(n), C.c_double(a_target), C.c_double(spread),
          C.c_uint64(seed), a00.ctypes.data_as(C.POINTER(C.c_double)),
          a01.ctypes.data_as(C.POINTER(C.c_double)))
    return InputMatrix(n, a00.view(np.complex128), a01.view(np.complex128))


def limbs_to_int(limbs, width_bits):
    v = 0
    for i in reversed(range(width_bits // 64)):
        v = (v << 64) | int(limbs[i])
    if v >> (width_bits - 1):
        v -= 1 << width_bits
    return v


def slice(m, width, frac_bits, k, lo, hi, threads=0):
    """Raw fixed-point class sums over prefix classes [lo, hi) of the top k mask bits.

    Returns (total_int, [class_int...], [class_sum_abs...]); value = int / 2^frac_bits.
    """
    threads = threads or os.cpu_count() or 1
    a00, a01, keep = _tri(m)
    n = hi - lo
    cl = (C.c_uint64 * (4 * n))()
    sa = (C.c_double * n)()
    tot = (C.c_uint64 * 4)()
    _call(lib().ref_slice, C.c_int(m.n_modes), a00, a01, C.c_int(width), C.c_int(frac_bits),
          C.c_int(k), C.c_uint64(lo), C.c_uint64(hi), C.c_int(threads), cl, sa, tot)
    per = [limbs_to_int(cl[4 * i:4 * i + 4], width) for i in range(n)]
    return limbs_to_int(tot, width), per, [sa[i] for i in range(n)]


def partial_sample(m, precision, nproc, rank_lo, nranks, threads):
    """Timed torontonian_partial over partition ranks (bounded CPU-baseline sample)."""
    p = {"128": 1, "256": 2}[str(precision)]
    a00, a01, keep = _tri(m)
    done = C.c_uint64()
    secs = C.c_double()
    _call(lib().ref_partial_sample, C.c_int(m.n_modes), a00, a01, C.c_int(p), C.c_int(nproc),
          C.c_int(rank_lo), C.c_int(nranks), C.c_int(threads), C.byref(done), C.byref(secs))
    return done.value, secs.value


def total_op_count(n):
    lo = C.c_uint64()
    hi = C.c_uint64()
    _call(lib().ref_total_op_count, C.c_int(n), C.byref(lo), C.byref(hi))
    return (hi.value << 64) | lo.value
