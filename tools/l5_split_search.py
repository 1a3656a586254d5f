"""Bank-conflict search for the split level-5 layout (engine.cu kL5Split): threads x and
x + 16 share parent pi(x); 128-bit shared-memory loads are served per 8-thread phase.  Scores
the parent trailing-block loads (A entries for threads 0-15, mirrors for 16-31), the
anti-diagonal loads and the pivot-row vector loads with the model of tools/l5_layout_search.py
and anneals the permutation.  usage: python tools/l5_split_search.py"""
import os
import random

HERE = os.path.dirname(os.path.abspath(__file__))
_src = open(os.path.join(HERE, "l5_layout_search.py")).read().split("def uw_cost")[0]
exec(_src.replace("print(", "(lambda *a, **k: None)("))  # node_off, base, A, cix, wavefronts, m, D


def split_cost(pi):
    tot = 0
    for C in range(8):
        for tt in (0, 1):
            i, j = A[2 * C + tt]
            kA, kB = cix(i, j), cix(D - 1 - j, D - 1 - i)
            tot += wavefronts([base[pi[t & 15]] + 2 * m - 1 + (kB if t >> 4 else kA) for t in range(32)])
    for a in range(4):
        tot += wavefronts([base[pi[t & 15]] + 2 * m - 1 + cix(a, D - 1 - a) for t in range(32)])
    for k in range(8):
        for off in (0, m):
            tot += wavefronts([pi[t & 15] * (2 * m + 1) + off + 2 + ((7 - k) if t >> 4 else k) for t in range(32)])
    return tot


if __name__ == "__main__":
    rng = random.Random(1)
    cur = list(range(16))
    cc = split_cost(cur)
    best = (cc, cur[:])
    print("ideal", (16 + 4 + 16) * 4, "identity", cc)
    for _ in range(200000):
        a, b = rng.randrange(16), rng.randrange(16)
        cur[a], cur[b] = cur[b], cur[a]
        c2 = split_cost(cur)
        if c2 <= cc or rng.random() < 0.001:
            cc = c2
            if cc < best[0]:
                best = (cc, cur[:])
        else:
            cur[a], cur[b] = cur[b], cur[a]
    print("best", best, hex(sum(p << (4 * i) for i, p in enumerate(best[1]))))
