"""TEST INFRASTRUCTURE ONLY: ctypes bindings to oracle/liboracle.so (tor_oracle.c).

The C restatement of the reference engine; pinned limb-exact against the reference's
golden values by tests/test_oracle.py.  Only tests/, __graft_entry__.smoke() and
bench.py's baseline legs use it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
_lib = None


class OracleError(RuntimeError):
    def __init__(self, status, code, msg, row=-1, mask=0):
        super().__init__(f"[{status}] {code}: {msg}")
        self.status, self.code, self.row, self.mask = status, code, row, mask


class _Err(C.Structure):
    _fields_ = [("status", C.c_int), ("code", C.c_char * 48), ("message", C.c_char * 160), ("row", C.c_int64),
                ("mask", C.c_uint64)]


class _Cfg(C.Structure):
    _fields_ = [("width_bits", C.c_int), ("frac_bits", C.c_uint), ("b_lower", C.c_int), ("b_upper", C.c_int),
                ("b_sgn", C.c_int), ("b_accum", C.c_int), ("a_repr", C.c_double), ("k_corr", C.c_double),
                ("alpha", C.c_double)]


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.or_binom.restype = C.c_uint64
        L.or_get_kth_mask.restype = C.c_uint64
        L.or_get_kth_mask.argtypes = [C.c_int, C.c_int, C.c_uint64]
        L.or_get_next_mask.restype = C.c_uint64
        L.or_get_next_mask.argtypes = [C.c_uint64]
        _lib = L
    return _lib


def _tri(m):
    a00, a01 = m.interleaved()
    return a00.ctypes.data_as(C.POINTER(C.c_double)), a01.ctypes.data_as(C.POINTER(C.c_double)), (a00, a01)


def _chk(st, e):
    if st:
        raise OracleError(st, e.code.decode(), e.message.decode(), e.row, e.mask)


def _cfg(c):
    return dict(width_bits=c.width_bits, frac_bits=c.frac_bits, b_lower=c.b_lower, b_upper=c.b_upper,
                b_sgn=c.b_sgn, b_accum=c.b_accum, a_repr=c.a_repr, k_corr=c.k_corr)


def limbs_to_int(limbs, width_bits):
    v = 0
    for i in reversed(range(width_bits // 64)):
        v = (v << 64) | int(limbs[i])
    if v >> (width_bits - 1):
        v -= 1 << width_bits
    return v


def select_precision(m, N=None, sig=3, alpha=0.5):
    a, b, keep = _tri(m)
    c, e = _Cfg(), _Err()
    _chk(lib().or_select_precision(m.n_modes, a, b, m.n_modes if N is None else N, sig, C.c_double(alpha),
                                   C.byref(c), C.byref(e)), e)
    return _cfg(c)


def force_width(m, width):
    a, b, keep = _tri(m)
    c, e = _Cfg(), _Err()
    _chk(lib().or_force_width(m.n_modes, a, b, width, C.byref(c), C.byref(e)), e)
    return _cfg(c)


def torontonian(m, precision="auto", threads=0):
    p = {"auto": 0, "128": 1, "256": 2}[str(precision)]
    a, b, keep = _tri(m)
    v = C.c_double()
    limbs = (C.c_uint64 * 4)()
    c, e = _Cfg(), _Err()
    _chk(lib().or_torontonian(m.n_modes, a, b, p, threads or os.cpu_count() or 1, C.byref(v), limbs, C.byref(c),
                              C.byref(e)), e)
    cfg = _cfg(c)
    return dict(value=v.value, raw=limbs_to_int(limbs, cfg["width_bits"]), raw_limbs=tuple(limbs), config=cfg)


def torontonian_reference(m):
    a, b, keep = _tri(m)
    v, e = C.c_double(), _Err()
    _chk(lib().or_torontonian_reference(m.n_modes, a, b, C.byref(v), C.byref(e)), e)
    return v.value


def slice(m, width, frac_bits, k, lo, hi, threads=0):
    a, b, keep = _tri(m)
    n = hi - lo
    cl = (C.c_uint64 * (4 * n))()
    sa = (C.c_double * n)()
    tot = (C.c_uint64 * 4)()
    e = _Err()
    _chk(lib().or_slice(m.n_modes, a, b, width, frac_bits, k, C.c_uint64(lo), C.c_uint64(hi),
                        threads or os.cpu_count() or 1, cl, sa, tot, C.byref(e)), e)
    return (limbs_to_int(tot, width), [limbs_to_int(cl[4 * i:4 * i + 4], width) for i in range(n)],
            [sa[i] for i in range(n)])


def partial_sample(m, width, seconds=10.0, threads=0):
    """Bounded timed sample of torontonian_partial-style work (CPU baseline, port kind)."""
    threads = threads or os.cpu_count() or 1
    a, b, keep = _tri(m)
    done, secs, e = C.c_uint64(), C.c_double(), _Err()
    nproc = 1 << 30
    _chk(lib().or_partial_sample(m.n_modes, a, b, width, nproc, 0, threads, threads, C.byref(done), C.byref(secs),
                                 C.byref(e)), e)
    rate = done.value / max(secs.value, 1e-9)
    nranks = max(threads, int(threads * rate * seconds / max(done.value, 1)))
    _chk(lib().or_partial_sample(m.n_modes, a, b, width, nproc, threads, nranks, threads, C.byref(done),
                                 C.byref(secs), C.byref(e)), e)
    return done.value, secs.value


def binom(n, k):
    return lib().or_binom(n, k)


def get_kth_mask(N, z, k):
    return lib().or_get_kth_mask(N, z, k)


def get_next_mask(mask):
    return lib().or_get_next_mask(mask)


def wide_mul(a: int, b: int, width: int, f: int) -> int:
    def limbs(v):
        v %= 1 << width
        return (C.c_uint64 * 4)(*[(v >> (64 * i)) & ((1 << 64) - 1) for i in range(4)])
    out = (C.c_uint64 * 4)()
    lib().or_wide_mul(limbs(a), limbs(b), width, C.c_uint(f), out)
    return limbs_to_int(out, width)


def wide_rsqrt(a: int, width: int, f: int) -> int:
    la = (C.c_uint64 * 4)(*[(a >> (64 * i)) & ((1 << 64) - 1) for i in range(4)])
    out = (C.c_uint64 * 4)()
    st = lib().or_wide_rsqrt(la, width, C.c_uint(f), out)
    if st:
        raise OracleError(st, "fixedpt/overflow" if st == -1 else "fixedpt/nonpositive", "rsqrt")
    return limbs_to_int(out, width)


__all__ = ["torontonian", "torontonian_reference", "select_precision", "force_width", "slice", "partial_sample",
           "binom", "get_kth_mask", "get_next_mask", "wide_mul", "wide_rsqrt", "np"]
