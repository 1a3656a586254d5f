"""Python mirror of the reference's ``torfp`` API for the hot path, over the C ABI.

Same names, argument meaning, result-dict keys and error behaviour as the
reference's pybind module (python/bindings.cpp:104-205, python/torfp/__init__.py),
but every evaluation runs on the GPU through ``libtor_b200.so``
(include/tor_capi.h).  There is no CPU fallback: a missing library or a missing
GPU raises (DeviceError / OSError), it never silently computes elsewhere.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from fractions import Fraction

import numpy as np

from . import errors as E
from .matrix import InputMatrix

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TOR_B200_LIB") or os.path.join(_PKG, "libtor_b200.so")

PREC_AUTO, PREC_DD, PREC_QD, PREC_FP64, PREC_FIXED128, PREC_FIXED256 = 0, 1, 2, 3, 4, 5
_PREC = {"auto": PREC_AUTO, "128": PREC_DD, "dd": PREC_DD, "256": PREC_QD, "qd": PREC_QD,
         "fp64": PREC_FP64, "64": PREC_FP64, "fixed128": PREC_FIXED128, "fixed256": PREC_FIXED256}
_MODE_NAME = {PREC_DD: "dd", PREC_QD: "qd", PREC_FP64: "fp64", PREC_FIXED128: "fixed128",
              PREC_FIXED256: "fixed256"}


class TorInput(C.Structure):
    _fields_ = [("n", C.c_int), ("a00_upper", C.POINTER(C.c_double)), ("a01_upper", C.POINTER(C.c_double))]


class TorPrecisionConfig(C.Structure):
    _fields_ = [("width_bits", C.c_int), ("frac_bits", C.c_uint), ("b_lower", C.c_int), ("b_upper", C.c_int),
                ("b_sgn", C.c_int), ("b_accum", C.c_int), ("a_repr", C.c_double), ("k_corr", C.c_double),
                ("alpha", C.c_double)]


class TorError(C.Structure):
    _fields_ = [("code", C.c_char * 48), ("message", C.c_char * 200), ("pivot_row", C.c_int64),
                ("subset_mask", C.c_uint64)]


class TorResult(C.Structure):
    _fields_ = [("value", C.c_double), ("mode", C.c_int), ("width_bits", C.c_int), ("nwords", C.c_int),
                ("words", C.c_double * 4), ("config", TorPrecisionConfig), ("term_count", C.c_uint64),
                ("mults", C.c_uint64), ("adds", C.c_uint64), ("recips", C.c_uint64), ("rsqrts", C.c_uint64),
                ("wall_seconds", C.c_double), ("device_ms", C.c_double), ("kernel_ms", C.c_double),
                ("devices", C.c_int), ("escalated", C.c_int), ("sum_abs_terms", C.c_double),
                ("cancellation_bits", C.c_double), ("bits_left", C.c_double), ("kernel_launches", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64), ("raw_limbs", C.c_uint64 * 4)]


class TorPartial(C.Structure):
    _fields_ = [("mode", C.c_int), ("class_bits", C.c_int), ("class_lo", C.c_uint64), ("class_hi", C.c_uint64),
                ("words", C.c_double * 4), ("sum_abs", C.c_double), ("term_count", C.c_uint64)]


class TorSchedule(C.Structure):
    _fields_ = [("prefix_jobs", C.c_uint64), ("blocks_per_sm", C.c_int), ("reserved", C.c_int)]


# every symbol include/tor_capi.h declares (checked by tests/test_capi.py)
EXPORTS = ("tor_abi_version", "tor_check_symmetries", "tor_check_dense", "tor_det_i_minus_a",
           "tor_select_precision", "tor_force_width", "tor_torontonian", "tor_torontonian_reference",
           "tor_torontonian_batch", "tor_torontonian_slice", "tor_torontonian_classes", "tor_torontonian_shard",
           "tor_fold_partials",
           "tor_probability", "tor_probability_modes", "tor_device_count", "tor_plan_create", "tor_plan_execute", "tor_plan_destroy",
           "tor_release_device_cache", "tor_load_matrix", "tor_save_matrix")

_lib = None


def lib():
    """Load libtor_b200.so (fails loudly when it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise OSError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                          "(python -m paper_2009_01177_b200._build)")
        L = C.CDLL(LIB_PATH)
        P = C.POINTER
        L.tor_torontonian.argtypes = [P(TorInput), C.c_int, P(C.c_int), C.c_int, P(TorResult), P(TorError)]
        L.tor_torontonian_reference.argtypes = [P(TorInput), P(C.c_double), P(TorError)]
        L.tor_torontonian_batch.argtypes = [P(TorInput), C.c_int, C.c_int, C.c_int, P(TorResult), P(TorError)]
        L.tor_torontonian_slice.argtypes = [P(TorInput), C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                            P(TorPartial), P(TorError)]
        L.tor_torontonian_classes.argtypes = [P(TorInput), C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                              P(TorSchedule), P(TorPartial), P(TorError)]
        L.tor_torontonian_shard.argtypes = [P(TorInput), C.c_int, C.c_int, C.c_int, C.c_int, P(TorPartial),
                                            P(TorError)]
        L.tor_fold_partials.argtypes = [P(TorPartial), C.c_int, P(TorInput), P(TorResult), P(TorError)]
        L.tor_select_precision.argtypes = [P(TorInput), C.c_int, C.c_int, C.c_double, P(TorPrecisionConfig),
                                           P(TorError)]
        L.tor_force_width.argtypes = [P(TorInput), C.c_int, P(TorPrecisionConfig), P(TorError)]
        L.tor_check_symmetries.argtypes = [P(TorInput), P(C.c_double), P(C.c_int), P(TorError)]
        L.tor_check_dense.argtypes = [C.c_int, P(C.c_double), P(C.c_double), P(C.c_int), P(TorError)]
        L.tor_det_i_minus_a.argtypes = [P(TorInput), P(C.c_double), P(TorError)]
        L.tor_probability.argtypes = [P(TorInput), C.c_uint64, C.c_int, C.c_int, P(C.c_double), P(TorError)]
        L.tor_probability_modes.argtypes = [P(TorInput), P(C.c_int), C.c_int, C.c_int, C.c_int, P(C.c_double),
                                            P(TorError)]
        L.tor_plan_create.argtypes = [P(TorInput), C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                      P(C.c_void_p), P(TorError)]
        L.tor_plan_execute.argtypes = [C.c_void_p, P(TorResult), P(TorError)]
        L.tor_plan_destroy.argtypes = [C.c_void_p]
        L.tor_plan_destroy.restype = None
        L.tor_load_matrix.argtypes = [C.c_char_p, C.c_size_t, P(C.c_int), P(C.c_int), P(C.c_double),
                                      P(C.c_double), C.c_size_t, P(TorError)]
        L.tor_save_matrix.argtypes = [P(TorInput), C.c_int, C.c_int, C.c_char_p, C.c_size_t, P(C.c_size_t),
                                      P(TorError)]
        L.tor_release_device_cache.argtypes = []
        L.tor_release_device_cache.restype = None
        _lib = L
    return _lib


class _In:
    """Keeps the interleaved arrays alive while the C side reads them."""

    def __init__(self, m: InputMatrix):
        self.a00, self.a01 = m.interleaved()
        self.s = TorInput(m.n_modes, self.a00.ctypes.data_as(C.POINTER(C.c_double)),
                          self.a01.ctypes.data_as(C.POINTER(C.c_double)))


def _check(status: int, err: TorError) -> None:
    if status:
        E.raise_for_status(status, err.code.decode(), err.message.decode(), int(err.pivot_row),
                           int(err.subset_mask))


def _prec(p) -> int:
    key = str(p).lower()
    if key not in _PREC:
        raise E.InvalidArgument("precision/range", "precision must be auto, 128, 256 or fp64")
    return _PREC[key]


def _cfg_dict(c: TorPrecisionConfig) -> dict:
    return dict(width_bits=c.width_bits, frac_bits=c.frac_bits, b_lower=c.b_lower, b_upper=c.b_upper,
                b_sgn=c.b_sgn, b_accum=c.b_accum, a_repr=c.a_repr, k_corr=c.k_corr)


def words_fraction(words) -> Fraction:
    return sum((Fraction(float(w)) for w in words), Fraction(0))


def raw_limbs(words, width_bits: int, frac_bits: int) -> tuple:
    """The multi-word value re-quantised at the reference's scaling 2^-frac_bits as
    two's-complement 64-bit limbs (low first, 4 entries like FixedValue::limbs)."""
    if width_bits not in (128, 256):
        return (0, 0, 0, 0)
    # exact integer arithmetic: every word is n / 2^k; common denominator 2^K
    parts = [float(w).as_integer_ratio() for w in words]
    K = max(d.bit_length() - 1 for _, d in parts)
    total = sum(n << (K - (d.bit_length() - 1)) for n, d in parts)
    # round(total * 2^f / 2^K), ties up (floor(v + 1/2))
    if frac_bits >= K:
        q = total << (frac_bits - K)
    else:
        sh = K - frac_bits
        q = (total + (1 << (sh - 1))) >> sh
    q %= 1 << width_bits
    return tuple((q >> (64 * i)) & ((1 << 64) - 1) if i < width_bits // 64 else 0 for i in range(4))


def _result_dict(r: TorResult, workers: int) -> dict:
    words = tuple(r.words[i] for i in range(4))
    cfg = _cfg_dict(r.config)
    return {
        # reference keys (bindings.cpp:69-85)
        "value": r.value,
        "raw_limbs": tuple(int(x) for x in r.raw_limbs),
        "width_bits": r.width_bits,
        "config": cfg,
        "term_count": r.term_count,
        "counters": dict(mults=r.mults, adds=r.adds, recips=r.recips, rsqrts=r.rsqrts),
        "wall_seconds": r.wall_seconds,
        "workers": workers,
        # engine extensions
        "mode": _MODE_NAME.get(r.mode, "?"),
        "words": words[: r.nwords] if r.nwords else words,
        "device_ms": r.device_ms,
        "kernel_ms": r.kernel_ms,
        "devices": r.devices,
        "escalated": bool(r.escalated),
        "sum_abs_terms": r.sum_abs_terms,
        "cancellation_bits": r.cancellation_bits,
        "bits_left": r.bits_left,
        "kernel_launches": r.kernel_launches,
        "h2d_bytes": r.h2d_bytes,
        "d2h_bytes": r.d2h_bytes,
    }


def torontonian(matrix: InputMatrix, precision="auto", workers: int = 0, devices=None) -> dict:
    """Tor(A) (torontonian.cpp:151-177) on the GPU.  ``precision``: "auto" | "128" | "256"
    (reference) or "fp64"; ``workers`` is accepted for drop-in compatibility (the
    engine's parallelism is the GPU); ``devices`` lists CUDA device ids."""
    inp = _In(matrix)
    devs = list(devices) if devices else [0]
    arr = (C.c_int * len(devs))(*devs)
    r = TorResult()
    err = TorError()
    _check(lib().tor_torontonian(C.byref(inp.s), _prec(precision), arr, len(devs), C.byref(r), C.byref(err)), err)
    return _result_dict(r, workers if workers > 0 else len(devs))


def torontonian_reference(matrix: InputMatrix) -> float:
    """fp64 oracle semantics (N <= 20) (torontonian.cpp:179-200), evaluated on the GPU."""
    inp = _In(matrix)
    v = C.c_double()
    err = TorError()
    _check(lib().tor_torontonian_reference(C.byref(inp.s), C.byref(v), C.byref(err)), err)
    return v.value


class BatchInputs:
    """`count` instances of equal N marshalled once for tor_torontonian_batch: the triangles
    stacked in two contiguous float64 arrays and the tor_input records built by numpy (no
    per-instance Python objects), reusable across calls."""

    def __init__(self, matrices):
        ms = list(matrices)
        if not ms:
            raise E.InvalidArgument("torontonian/range", "empty batch")
        self.n = ms[0].n_modes
        self.count = len(ms)
        self.array = (TorInput * self.count)()
        if any(m.n_modes != self.n for m in ms):  # mixed N: the C side reports it
            self._keep = [_In(m) for m in ms]
            for i, k in enumerate(self._keep):
                self.array[i] = k.s
            return
        self.a00 = np.ascontiguousarray(np.stack([np.asarray(m.a00, np.complex128) for m in ms]).view(np.float64))
        self.a01 = np.ascontiguousarray(np.stack([np.asarray(m.a01, np.complex128) for m in ms]).view(np.float64))
        rec = np.frombuffer(self.array, dtype=np.dtype({"names": ["n", "a00", "a01"], "formats": ["<i4", "<u8", "<u8"],
                                                        "offsets": [0, 8, 16], "itemsize": C.sizeof(TorInput)}))
        stride = self.a00.shape[1] * 8
        rec["n"] = self.n
        rec["a00"] = self.a00.ctypes.data + stride * np.arange(self.count, dtype=np.uint64)
        rec["a01"] = self.a01.ctypes.data + stride * np.arange(self.count, dtype=np.uint64)


_RESULT_DTYPE = None


def _result_dtype():
    global _RESULT_DTYPE
    if _RESULT_DTYPE is None:
        names, fmts, offs = [], [], []
        for name in ("value", "mode", "width_bits", "nwords", "words", "term_count", "device_ms", "kernel_ms",
                     "escalated", "sum_abs_terms", "cancellation_bits", "bits_left", "kernel_launches"):
            f = getattr(TorResult, name)
            names.append(name)
            offs.append(f.offset)
            fmts.append({"words": ("<f8", (4,)), "mode": "<i4", "width_bits": "<i4", "nwords": "<i4",
                         "escalated": "<i4", "term_count": "<u8", "kernel_launches": "<u8"}.get(name, "<f8"))
        _RESULT_DTYPE = np.dtype({"names": names, "formats": fmts, "offsets": offs,
                                  "itemsize": C.sizeof(TorResult)})
    return _RESULT_DTYPE


def torontonian_batch_raw(batch: BatchInputs, precision="fp64", device: int = 0) -> np.ndarray:
    """tor_torontonian_batch on pre-marshalled inputs; returns a numpy structured array view
    of the tor_result records (fields value, words, sum_abs_terms, mode, escalated, ...)."""
    res = (TorResult * batch.count)()
    err = TorError()
    _check(lib().tor_torontonian_batch(batch.array, batch.count, _prec(precision), device, res, C.byref(err)), err)
    return np.frombuffer(res, dtype=_result_dtype())


def torontonian_batch(matrices, precision="fp64", device: int = 0) -> list[dict]:
    batch = matrices if isinstance(matrices, BatchInputs) else BatchInputs(matrices)
    res = (TorResult * batch.count)()
    err = TorError()
    _check(lib().tor_torontonian_batch(batch.array, batch.count, _prec(precision), device, res, C.byref(err)), err)
    return [_result_dict(res[i], 1) for i in range(batch.count)]


def torontonian_slice(matrix: InputMatrix, precision, class_bits: int, class_lo: int, class_hi: int,
                      device: int = 0) -> dict:
    inp = _In(matrix)
    p = TorPartial()
    err = TorError()
    _check(lib().tor_torontonian_slice(C.byref(inp.s), _prec(precision), class_bits, class_lo, class_hi, device,
                                       C.byref(p), C.byref(err)), err)
    return _partial_dict(p)


def torontonian_classes(matrix: InputMatrix, precision, class_bits: int, class_lo: int, class_hi: int,
                        device: int = 0, prefix_jobs: int = 0, blocks_per_sm: int = 0) -> list[dict]:
    """One partial per prefix class of [class_lo, class_hi) from one device pass
    (tor_torontonian_classes); ``prefix_jobs`` / ``blocks_per_sm`` are the schedule hints
    (0 = default)."""
    inp = _In(matrix)
    cnt = class_hi - class_lo
    arr = (TorPartial * max(cnt, 1))()
    sch = TorSchedule(prefix_jobs, blocks_per_sm, 0)
    err = TorError()
    _check(lib().tor_torontonian_classes(C.byref(inp.s), _prec(precision), class_bits, class_lo, class_hi, device,
                                         C.byref(sch), arr, C.byref(err)), err)
    return [_partial_dict(arr[i]) for i in range(cnt)]


def torontonian_shard(matrix: InputMatrix, precision, rank: int, world: int, device: int = 0) -> dict:
    inp = _In(matrix)
    p = TorPartial()
    err = TorError()
    _check(lib().tor_torontonian_shard(C.byref(inp.s), _prec(precision), rank, world, device, C.byref(p),
                                       C.byref(err)), err)
    return _partial_dict(p)


def _partial_dict(p: TorPartial) -> dict:
    return dict(mode=p.mode, class_bits=p.class_bits, class_lo=p.class_lo, class_hi=p.class_hi,
                words=tuple(p.words[i] for i in range(4)), sum_abs=p.sum_abs, term_count=p.term_count)


def partial_to_array(p: dict) -> np.ndarray:
    """Shard partial as 10 float64 (for torch.distributed all_gather)."""
    return np.array([p["mode"], p["class_bits"], p["class_lo"], p["class_hi"], *p["words"], p["sum_abs"],
                     p["term_count"]], dtype=np.float64)


def array_to_partial(a) -> dict:
    a = [float(x) for x in a]
    return dict(mode=int(a[0]), class_bits=int(a[1]), class_lo=int(a[2]), class_hi=int(a[3]),
                words=tuple(a[4:8]), sum_abs=a[8], term_count=int(a[9]))


def fold_partials(parts: list[dict], matrix: InputMatrix) -> dict:
    parts = sorted(parts, key=lambda p: p["class_lo"])
    arr = (TorPartial * len(parts))()
    for i, p in enumerate(parts):
        arr[i] = TorPartial(p["mode"], p["class_bits"], p["class_lo"], p["class_hi"], (C.c_double * 4)(*p["words"]),
                            p["sum_abs"], p["term_count"])
    inp = _In(matrix)
    r = TorResult()
    err = TorError()
    _check(lib().tor_fold_partials(arr, len(parts), C.byref(inp.s), C.byref(r), C.byref(err)), err)
    return _result_dict(r, len(parts))


def select_precision(matrix: InputMatrix, n_modes: int | None = None, sig_decimal_digits: int = 3,
                     alpha: float = 0.5) -> dict:
    """select_precision (precision.cpp:80-121), host port with identical decisions."""
    inp = _In(matrix)
    c = TorPrecisionConfig()
    err = TorError()
    N = matrix.n_modes if n_modes is None else n_modes
    _check(lib().tor_select_precision(C.byref(inp.s), N, sig_decimal_digits, alpha, C.byref(c), C.byref(err)), err)
    return _cfg_dict(c)


def force_width(matrix: InputMatrix, width_bits: int) -> dict:
    inp = _In(matrix)
    c = TorPrecisionConfig()
    err = TorError()
    _check(lib().tor_force_width(C.byref(inp.s), width_bits, C.byref(c), C.byref(err)), err)
    return _cfg_dict(c)


def det_i_minus_a(matrix: InputMatrix) -> float:
    inp = _In(matrix)
    v = C.c_double()
    err = TorError()
    _check(lib().tor_det_i_minus_a(C.byref(inp.s), C.byref(v), C.byref(err)), err)
    return v.value


def probability(matrix: InputMatrix, pattern_bits, workers: int = 0, precision="auto",
                device: int = 0) -> float:
    """p(S) = Tor(A_S) sqrt(det(I - A)) (torontonian.cpp:202-209).  pattern_bits: an int
    (bit k = mode k, the reference's ClickPattern) or a sequence of mode indices (no 64-mode
    limit: tor_probability_modes)."""
    inp = _In(matrix)
    v = C.c_double()
    err = TorError()
    if isinstance(pattern_bits, (int, np.integer)):
        _check(lib().tor_probability(C.byref(inp.s), int(pattern_bits), _prec(precision), device, C.byref(v),
                                     C.byref(err)), err)
    else:
        modes = sorted(int(k) for k in pattern_bits)
        arr = (C.c_int * max(len(modes), 1))(*modes)
        _check(lib().tor_probability_modes(C.byref(inp.s), arr, len(modes), _prec(precision), device, C.byref(v),
                                           C.byref(err)), err)
    return v.value


def probability_reference(matrix: InputMatrix, pattern_bits: int) -> float:
    return probability(matrix, pattern_bits, precision="fp64")


class Plan:
    """Device-resident evaluation (tor_plan_*): inputs uploaded once, execute() reruns the
    whole device pipeline.  Used by bench.py for the HBM-resident throughput figure."""

    def __init__(self, matrix: InputMatrix, precision, class_bits: int = 0, class_lo: int = 0,
                 class_hi: int = 1, device: int = 0):
        self._inp = _In(matrix)
        self._h = C.c_void_p()
        err = TorError()
        _check(lib().tor_plan_create(C.byref(self._inp.s), _prec(precision), class_bits, class_lo, class_hi,
                                     device, C.byref(self._h), C.byref(err)), err)

    def execute(self) -> dict:
        r = TorResult()
        err = TorError()
        _check(lib().tor_plan_execute(self._h, C.byref(r), C.byref(err)), err)
        return _result_dict(r, 1)

    def close(self) -> None:
        if self._h:
            lib().tor_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_count() -> int:
    return lib().tor_device_count()


def release_device_cache() -> None:
    """Free the device memory pooled between calls (tor_release_device_cache)."""
    lib().tor_release_device_cache()


def load_matrix_bytes(b: bytes) -> InputMatrix:
    """GBSA bytes -> InputMatrix through tor_load_matrix (load_matrix_file's format sniffing,
    matrix_io.cpp:253-263)."""
    b = bytes(b)
    n, qb = C.c_int(), C.c_int()
    err = TorError()
    _check(lib().tor_load_matrix(b, len(b), C.byref(n), C.byref(qb), None, None, 0, C.byref(err)), err)
    t = n.value * (n.value + 1) // 2
    a00 = np.zeros(2 * t)
    a01 = np.zeros(2 * t)
    P = C.POINTER(C.c_double)
    _check(lib().tor_load_matrix(b, len(b), C.byref(n), C.byref(qb), a00.ctypes.data_as(P), a01.ctypes.data_as(P), t,
                                 C.byref(err)), err)
    return InputMatrix(n.value, a00.view(np.complex128), a01.view(np.complex128), quant_bits=qb.value)


def save_matrix_bytes(matrix: InputMatrix, format: str = "text", quant_bits: int = 16) -> bytes:
    """InputMatrix -> GBSA bytes through tor_save_matrix (save_matrix, matrix_io.cpp:109-143)."""
    if format not in ("text", "binary"):
        raise E.InvalidArgument("matrixio/format", "format must be 'text' or 'binary'")
    inp = _In(matrix)
    size = C.c_size_t()
    err = TorError()
    fmt = 1 if format == "binary" else 0
    _check(lib().tor_save_matrix(C.byref(inp.s), fmt, quant_bits, None, 0, C.byref(size), C.byref(err)), err)
    buf = C.create_string_buffer(size.value)
    _check(lib().tor_save_matrix(C.byref(inp.s), fmt, quant_bits, buf, size.value, C.byref(size), C.byref(err)), err)
    return buf.raw[: size.value]
