"""Instance data model and GBSA text/binary file formats (host side).

Mirrors the reference data model so that callers of ``torfp`` find the same
objects here:

* ``InputMatrix``: block-symmetric A = [[A00, A01], [conj A01, conj A00]] over
  N modes, stored as the two upper triangles, row-major, index
  ``i*n - i(i+1)/2 + j`` (reference ``matrix_io.hpp:18-26``, ``linalg.hpp:32-35``).
* ``from_dense`` with the 1e-12 symmetry gate (``bindings.cpp:26-47``,
  ``matrix_io.cpp:285-305``).
* ``to_dense`` (``matrix_io.cpp:265-283``), ``extract_submatrix``
  (``matrix_io.cpp:360-382``).
* GBSA text (lossless, ``matrix_io.cpp:116-128`` / ``:195-229``) and binary
  (quantised, ``matrix_io.cpp:131-146`` / ``:150-193``) formats.

Pure numpy; no device code lives here.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from .errors import InvalidArgument, TorfpError

SYMMETRY_TOL = 1e-12  # matrix_io.hpp:62


def tri_size(n: int) -> int:
    return n * (n + 1) // 2


def tri_index(n: int, i: int, j: int) -> int:
    """Packed upper-triangle index, i <= j (linalg.hpp:32-35)."""
    return i * n - i * (i + 1) // 2 + j


def _upper(dense_block: np.ndarray) -> np.ndarray:
    n = dense_block.shape[0]
    iu = np.triu_indices(n)
    return np.ascontiguousarray(dense_block[iu], dtype=np.complex128)


@dataclass
class InputMatrix:
    """Two complex upper triangles (A00 Hermitian, A01 symmetric)."""

    n_modes: int
    a00: np.ndarray  # complex128, tri_size(n)
    a01: np.ndarray  # complex128, tri_size(n)
    quant_bits: int = 0
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        self.a00 = np.ascontiguousarray(self.a00, dtype=np.complex128)
        self.a01 = np.ascontiguousarray(self.a01, dtype=np.complex128)
        if self.n_modes < 1:
            raise InvalidArgument("matrixio/dim", "matrix has no modes")
        t = tri_size(self.n_modes)
        if self.a00.shape != (t,) or self.a01.shape != (t,):
            raise InvalidArgument("matrixio/dim", "triangle storage size mismatch")

    # a00_at / a01_at: matrix_io.cpp:80-88
    def a00_full(self) -> np.ndarray:
        n = self.n_modes
        m = np.zeros((n, n), dtype=np.complex128)
        iu = np.triu_indices(n)
        m[iu] = self.a00
        il = (iu[1], iu[0])
        m[il] = np.conj(self.a00)
        # diagonal: keep the stored value (the reference returns a00[tri(i,i)] for i == j)
        m[np.diag_indices(n)] = self.a00[[tri_index(n, i, i) for i in range(n)]]
        return m

    def a01_full(self) -> np.ndarray:
        n = self.n_modes
        m = np.zeros((n, n), dtype=np.complex128)
        iu = np.triu_indices(n)
        m[iu] = self.a01
        m[(iu[1], iu[0])] = self.a01
        return m

    def to_dense(self) -> np.ndarray:
        """Full 2N x 2N matrix [[A00, A01], [conj A01, conj A00]] (matrix_io.cpp:265-283)."""
        a00 = self.a00_full()
        a01 = self.a01_full()
        return np.block([[a00, a01], [np.conj(a01), np.conj(a00)]])

    def interleaved(self) -> tuple[np.ndarray, np.ndarray]:
        """(re, im) interleaved float64 triangles, the C-ABI layout (include/tor_capi.h)."""
        return (np.ascontiguousarray(self.a00.view(np.float64)),
                np.ascontiguousarray(self.a01.view(np.float64)))

    def save(self, path: str, format: str = "binary", bits: int = 16) -> None:
        data = save_matrix(self, "text" if format == "text" else "binary", bits)
        with open(path, "wb") as f:
            f.write(data)

    def __repr__(self) -> str:
        return f"<InputMatrix of {self.n_modes} modes>"


def symmetry_report(dense: np.ndarray) -> dict:
    """check_symmetries (matrix_io.cpp:285-305): max element deviations vs 1e-12."""
    dense = np.asarray(dense, dtype=np.complex128)
    d = dense.shape[0]
    if dense.ndim != 2 or dense.shape[1] != d or d < 2 or d % 2:
        raise InvalidArgument("matrixio/dim", "dense matrix must be 2N x 2N")
    n = d // 2
    herm = float(np.max(np.abs(dense - np.conj(dense.T))))
    a01 = dense[:n, n:]
    sym = float(np.max(np.abs(a01 - a01.T)))
    blk = float(np.max(np.abs(dense[:n, :n] - np.conj(dense[n:, n:]))))
    ok = herm <= SYMMETRY_TOL and sym <= SYMMETRY_TOL and blk <= SYMMETRY_TOL
    return {"hermitian_dev": herm, "a01_sym_dev": sym, "block_conj_dev": blk,
            "tolerance": SYMMETRY_TOL, "pass": bool(ok)}


def check_symmetries(m: InputMatrix) -> dict:
    return symmetry_report(m.to_dense())


def from_dense(dense) -> InputMatrix:
    """Build an instance from a full 2N x 2N array, symmetries checked (bindings.cpp:26-47)."""
    arr = np.asarray(dense, dtype=np.complex128)
    if arr.ndim != 2 or arr.shape[0] != arr.shape[1] or arr.shape[0] % 2 or arr.shape[0] == 0:
        raise InvalidArgument("matrixio/dim", "expected a square 2N x 2N array, N >= 1")
    if not symmetry_report(arr)["pass"]:
        raise TorfpError("torontonian/symmetry", "input violates the block symmetries beyond 1e-12")
    n = arr.shape[0] // 2
    return InputMatrix(n, _upper(arr[:n, :n]), _upper(arr[:n, n:]))


def extract_submatrix(a: InputMatrix, pattern_bits: int) -> InputMatrix:
    """Principal submatrix over clicked modes; bit k = mode k (matrix_io.cpp:360-382)."""
    sel = [k for k in range(a.n_modes) if (pattern_bits >> k) & 1]
    if pattern_bits >> a.n_modes:
        raise InvalidArgument("matrixio/dim", "pattern mode count mismatch")
    if not sel:
        raise InvalidArgument("matrixio/pattern", "empty click pattern")
    return select_modes(a, sel)


def select_modes(a: InputMatrix, sel) -> InputMatrix:
    sel = np.asarray(sel, dtype=np.int64)
    a00 = a.a00_full()[np.ix_(sel, sel)]
    a01 = a.a01_full()[np.ix_(sel, sel)]
    return InputMatrix(len(sel), _upper(a00), _upper(a01), quant_bits=a.quant_bits)


# ----------------------------------------------------------------- formats --


def quantize(x: float, bits: int) -> int:
    """Midpoint lattice, half away from zero, clamped (matrix_io.cpp:92-101)."""
    if bits not in (16, 32):
        raise InvalidArgument("matrixio/bits", "quantization width must be 16 or 32")
    if not abs(x) < 1.0:
        raise InvalidArgument("matrixio/range", "quantization requires |x| < 1")
    scale = math.ldexp(1.0, bits - 1)
    v = x * scale
    q = int(math.floor(abs(v) + 0.5)) * (1 if v >= 0 else -1)
    lim = int(scale) - 1
    return max(-lim, min(lim, q))


def dequantize(q: int, bits: int) -> float:
    if bits not in (16, 32):
        raise InvalidArgument("matrixio/bits", "quantization width must be 16 or 32")
    return float(q) * math.ldexp(1.0, -(bits - 1))


def save_matrix(a: InputMatrix, format: str = "text", quant_bits: int = 16) -> bytes:
    """save_matrix (matrix_io.cpp:109-143) through the C ABI (tor_save_matrix)."""
    from .api import save_matrix_bytes
    return save_matrix_bytes(a, format, quant_bits)


def load_matrix_bytes(b: bytes) -> InputMatrix:
    """Format sniffed from the magic (matrix_io.cpp:253-263), through the C ABI
    (tor_load_matrix)."""
    from .api import load_matrix_bytes as _load
    return _load(b)


def load_matrix(path: str) -> InputMatrix:
    if not os.path.exists(path):
        raise TorfpError("matrixio/io", f"cannot open for reading: {path}")
    with open(path, "rb") as f:
        return load_matrix_bytes(f.read())
