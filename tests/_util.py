"""Shared tolerance helpers for parity tests (exact rational comparisons)."""
from __future__ import annotations

from fractions import Fraction

# Per-mode absolute tolerance relative to sum |terms|; the alternating
# sum cancels, so the bound is against sum|t|, not |Tor|.
EPS = {"fp64": 2.0 ** -44, "dd": 2.0 ** -88, "qd": 2.0 ** -180}


def words_value(words) -> Fraction:
    return sum((Fraction(float(w)) for w in words), Fraction(0))


def fixed_value(raw: str | int, frac_bits: int) -> Fraction:
    return Fraction(int(raw), 1 << int(frac_bits))


def abs_err(a, b) -> float:
    return float(abs(Fraction(a) - Fraction(b)))


def within(got, want, sum_abs: float, mode: str) -> tuple[bool, float]:
    """|got - want| <= eps_mode * sum|t|; returns (ok, error in units of sum|t|)."""
    err = abs_err(got, want)
    rel = err / sum_abs if sum_abs else err
    return rel <= EPS[mode], rel
