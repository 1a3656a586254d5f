"""Seeded synthetic Gaussian-boson-sampling instances for BASELINE.json's configs.

There is no public benchmark suite for this path; these seeded pure states
stand in for one.  Recipe:

* rng = numpy.random.default_rng([2026, cfg]) draws the Haar unitary and the
  squeezing; default_rng([2026, cfg, item]) draws the click set S of item.
* Haar U: QR of (N(0,1) + i N(0,1))/sqrt 2, phase-fixed U diag(R_ii/|R_ii|).
* Pure state: B = U diag(-tanh r) U^T, symmetrised (B + B^T)/2; the
  O-matrix of the full state is [[0, B], [conj B, 0]] in (a, a^dagger) order
  (O = I - Q^{-1}, Q the Husimi covariance), i.e. InputMatrix(A00=0, A01=B).
* O_S keeps rows/columns {j, m+j : j in S}, S sorted ascending.

The generated instances are committed under tests/golden/ (GBSA text,
lossless) so every machine reads identical doubles regardless of LAPACK.
"""
from __future__ import annotations

import os

import numpy as np

from .matrix import InputMatrix, _upper, load_matrix, save_matrix, select_modes

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                          "tests", "golden")

# cfg id -> (m modes, squeezing spec, |S|, items, precision of record)
CONFIGS = {
    1: dict(m=32, r=("fixed", 1.0), n=16, items=1, select="first", mode="fp64"),
    2: dict(m=50, r=("uniform", 0.6, 1.2), n=20, items=1, select="random", mode="dd"),
    3: dict(m=100, r=("fixed", 1.0), n=16, items=4096, select="random", mode="fp64+dd"),
    4: dict(m=100, r=("uniform", 0.8, 1.6), n=32, items=1, select="random", mode="qd"),
    5: dict(m=100, r=("fixed", 1.2), n=40, items=1, select="random", mode="dd"),
}


def haar_unitary(rng: np.random.Generator, m: int) -> np.ndarray:
    z = (rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(2.0)
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    return q * (d / np.abs(d))[None, :]


def full_state(cfg: int) -> InputMatrix:
    """The m-mode pure state of config `cfg` as an InputMatrix (A00 = 0, A01 = B)."""
    c = CONFIGS[cfg]
    m = c["m"]
    rng = np.random.default_rng([2026, cfg])
    u = haar_unitary(rng, m)
    spec = c["r"]
    if spec[0] == "fixed":
        r = np.full(m, spec[1])
    else:
        r = rng.uniform(spec[1], spec[2], m)
    b = u @ np.diag(-np.tanh(r)) @ u.T
    b = (b + b.T) / 2.0
    a00 = np.zeros((m, m), dtype=np.complex128)
    return InputMatrix(m, _upper(a00), _upper(b))


def click_set(cfg: int, item: int = 0) -> list[int]:
    c = CONFIGS[cfg]
    if c["select"] == "first":
        return list(range(c["n"]))
    rng = np.random.default_rng([2026, cfg, item])
    return sorted(int(x) for x in rng.choice(c["m"], c["n"], replace=False))


def instance(cfg: int, item: int = 0, state: InputMatrix | None = None) -> InputMatrix:
    st = state if state is not None else full_state(cfg)
    return select_modes(st, click_set(cfg, item))


def pattern_bits(sel) -> int:
    """Click pattern bits (bit k = mode k, matrix_io.hpp:29-34)."""
    v = 0
    for k in sel:
        v |= 1 << int(k)
    return v


# ------------------------------------------------------------ committed ----
def golden_path(name: str) -> str:
    return os.path.join(GOLDEN_DIR, name)


def load_config_instance(cfg: int, item: int = 0) -> InputMatrix:
    """Committed O_S of config `cfg` (cfg3: extracted from the committed full state)."""
    if cfg == 3:
        st = load_matrix(golden_path("cfg3_state.gbsa.txt"))
        return select_modes(st, click_set(3, item))
    return load_matrix(golden_path(f"cfg{cfg}.gbsa.txt"))


def load_cfg3_batch(count: int = 4096) -> list[InputMatrix]:
    st = load_matrix(golden_path("cfg3_state.gbsa.txt"))
    return [select_modes(st, click_set(3, i)) for i in range(count)]


def write_config_fixtures() -> None:
    os.makedirs(GOLDEN_DIR, exist_ok=True)
    for cfg in (1, 2, 4, 5):
        with open(golden_path(f"cfg{cfg}.gbsa.txt"), "wb") as f:
            f.write(save_matrix(instance(cfg), "text"))
    with open(golden_path("cfg3_state.gbsa.txt"), "wb") as f:
        f.write(save_matrix(full_state(3), "text"))


# --------------------------------------------------- reference generator ----
_M64 = (1 << 64) - 1


def _rotl(x: int, k: int) -> int:
    return ((x << k) | (x >> (64 - k))) & _M64


class _Xoshiro256:
    """xoshiro256** seeded by splitmix64 expansion (matrix_io.cpp:18-47)."""

    def __init__(self, seed: int):
        x = seed & _M64
        self.s = []
        for _ in range(4):
            x = (x + 0x9E3779B97F4A7C15) & _M64
            z = x
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
            self.s.append(z ^ (z >> 31))

    def next(self) -> int:
        s = self.s
        result = (_rotl((s[1] * 5) & _M64, 7) * 9) & _M64
        t = (s[1] << 17) & _M64
        s[2] ^= s[0]
        s[3] ^= s[1]
        s[1] ^= s[2]
        s[0] ^= s[3]
        s[2] ^= t
        s[3] = _rotl(s[3], 45)
        return result

    def uniform_pm1(self) -> float:
        return float(self.next() >> 11) * 2.0 ** -52 - 1.0


def generate_instance(n_modes: int, a_target: float, spread: float, seed: int) -> InputMatrix:
    """Reference synthetic instance A = delta I + gamma H (matrix_io.cpp:307-358)."""
    from .errors import InvalidArgument
    from .matrix import tri_index, tri_size
    if n_modes < 1:
        raise InvalidArgument("matrixio/dim", "need at least one mode")
    if not (0.0 < a_target < 1.0):
        raise InvalidArgument("matrixio/range", "a_target must lie in (0,1)")
    if not (spread >= 0.0 and a_target - spread > 0.0 and a_target + spread < 1.0):
        raise InvalidArgument("matrixio/range", "spread leaves (0,1)")
    rng = _Xoshiro256(seed)
    n = n_modes
    t = tri_size(n)
    h00 = [0j] * t
    h01 = [0j] * t
    for i in range(n):
        for j in range(i, n):
            re = rng.uniform_pm1()
            im = 0.0 if i == j else rng.uniform_pm1()
            h00[tri_index(n, i, j)] = complex(re, im)
    for i in range(n):
        for j in range(i, n):
            re = rng.uniform_pm1()
            im = rng.uniform_pm1()
            h01[tri_index(n, i, j)] = complex(re, im)

    def a00_at(i, j):
        return h00[tri_index(n, i, j)] if i <= j else h00[tri_index(n, j, i)].conjugate()

    def a01_at(i, j):
        return h01[tri_index(n, i, j)] if i <= j else h01[tri_index(n, j, i)]

    max_row = 0.0
    for i in range(n):
        row = 0.0
        for j in range(n):
            row += abs(a00_at(i, j)) + abs(a01_at(i, j))
        max_row = max(max_row, row)
    gamma = 0.9 * spread / max_row if (spread > 0.0 and max_row > 0.0) else 0.0
    a00 = np.empty(t, dtype=np.complex128)
    a01 = np.empty(t, dtype=np.complex128)
    for i in range(n):
        for j in range(i, n):
            idx = tri_index(n, i, j)
            v = complex(gamma * h00[idx].real, gamma * h00[idx].imag)
            if i == j:
                v = complex(v.real + a_target, v.imag)
            a00[idx] = v
            a01[idx] = complex(gamma * h01[idx].real, gamma * h01[idx].imag)
    return InputMatrix(n, a00, a01)
