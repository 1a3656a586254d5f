"""Subset enumeration, work partitioning and operation-count formulas (host side).

Reference counterparts: subsets.hpp:13-46 / subsets.cpp:13-88 (binom, get_kth_mask,
get_next_mask, partition) and flops.cpp:9-31 (Eq. 7 / Eq. 8).  The GPU engine does not
use the popcount-class partition -- it splits the subset space into prefix classes
(top k mask bits, ``prefix_classes``) -- but callers of the reference API find the same
functions here.  Masks: bit N-1-j = mode j.
"""
from __future__ import annotations

import math

from .errors import InvalidArgument

_MAXN = 62


def binom(n: int, k: int) -> int:
    if n < 0 or k < 0 or k > n:
        raise InvalidArgument("subsets/range", "binom requires 0 <= k <= n")
    if n > _MAXN:
        raise InvalidArgument("subsets/overflow", "binom limited to n <= 62 (64-bit exact)")
    return math.comb(n, k)


def get_kth_mask(N: int, z: int, k: int) -> int:
    """k-th N-bit mask of popcount z in descending numeric order."""
    if N < 1 or N > _MAXN or z < 1 or z > N:
        raise InvalidArgument("subsets/range", "get_kth_mask requires 1 <= z <= N <= 62")
    if k >= binom(N, z):
        raise InvalidArgument("subsets/range", "get_kth_mask rank out of range")
    m, rem = 0, z
    for p in range(N - 1, -1, -1):
        if rem == 0:
            break
        cnt = binom(p, rem - 1)
        if k < cnt:
            m |= 1 << p
            rem -= 1
        else:
            k -= cnt
    return m


def get_next_mask(mask: int) -> int:
    """Descending-order successor with equal popcount; 0 at the end of the class."""
    t = 0
    while (mask >> t) & 1:
        t += 1
    x = mask - ((1 << t) - 1)
    if x == 0:
        return 0
    p = (x & -x).bit_length() - 1
    return x - (1 << (p - t - 1))


def partition(modes: int, rank: int, nproc: int) -> list[tuple[int, int, int]]:
    """Per-|Z| (start_mask, end_mask, count) slices of one worker (subsets.cpp:66-88)."""
    if modes < 1 or modes > _MAXN:
        raise InvalidArgument("subsets/range", "partition requires 1 <= N <= 62")
    if nproc < 1 or rank < 0 or rank >= nproc:
        raise InvalidArgument("subsets/range", "partition requires 0 <= rank < nproc")
    out = []
    for z in range(1, modes + 1):
        total = binom(modes, z)
        lo = total * rank // nproc
        hi = total * (rank + 1) // nproc
        cnt = hi - lo
        start = get_kth_mask(modes, z, lo) if cnt else 0
        end = get_kth_mask(modes, z, hi) if (cnt and hi < total) else 0
        out.append((start, end, cnt))
    return out


def prefix_classes(N: int, rank: int, world: int) -> tuple[int, int, int]:
    """The engine's shard of rank/world: (class_bits, class_lo, class_hi) over the top
    log2(world) mask bits (world a power of two)."""
    if world < 1 or world & (world - 1) or not 0 <= rank < world:
        raise InvalidArgument("torontonian/shard", "world must be a power of two and 0 <= rank < world")
    k = world.bit_length() - 1
    if k > N:
        raise InvalidArgument("torontonian/shard", "more shards than prefix classes")
    return k, rank, rank + 1


def factorization_op_count(dim: int) -> int:
    """(4d^3 + 3d^2 - 4d)/3 (flops.cpp:9-13, PAPER Eq. 7)."""
    if dim < 1 or dim > 1000:
        raise InvalidArgument("subsets/range", "dimension out of range")
    return (4 * dim ** 3 + 3 * dim ** 2 - 4 * dim) // 3


def total_op_count(n_modes: int) -> int:
    """Sum_z C(n,z) * factorization_op_count(2z) (flops.cpp:15-31, PAPER Eq. 8)."""
    if n_modes < 1 or n_modes > 60:
        raise InvalidArgument("subsets/range", "mode count must be in [1, 60]")
    return sum(math.comb(n_modes, z) * factorization_op_count(2 * z) for z in range(1, n_modes + 1))
