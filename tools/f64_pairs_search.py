"""Bank-conflict model and layout search for the fp64 fan-out with per-parent lane groups
(FanLevel::run_pairs) and the lane subtrees' level-5 reads (8-byte words in shared memory).

Model (matches the ncu wavefronts of the first version to within rounding): 8- and 16-byte
accesses are served per 16- / 8-lane phase; a phase costs the max over the bank slots of the
number of DISTINCT addresses in the slot (identical addresses are broadcast).  Per leaf, every fan-out level runs its pivot loads, pivot-row vector
loads and (u, w)-pair stores, then NS items (table word, source, two pairs, store); the
lane subtrees read their level-5 node states at compile-time offsets from the node bases.

Searched: level base pads, child stride adds (WarpSmem::lvl_pad / buf_stride for fp64), the
lane -> (parent, group lane) map of each level (parent-major or interleaved), and the pair
strides (m + 1..8 pairs).  usage: python tools/f64_pairs_search.py [iterations]"""
import collections
import random
import sys

Q0, FAN = 10, 5


def tri(d):
    return d * (d + 1) // 2


def tri_ix(d, i, j):
    return i * d - (i * (i + 1)) // 2 + j


def layout(pads, adds):
    def stride(e):
        return tri(2 * (Q0 - e)) + adds[e - 1]

    def lvl_off(e):
        o = tri(2 * Q0)
        for x in range(1, e):
            o += pads[x - 1] + (1 << (x - 1)) * stride(x)
        return 0 if e == 0 else o + (pads[e - 1] if e <= FAN else 0)

    def node_off(e, c):
        if c == 0:
            return tri_ix(2 * Q0, 2 * e, 2 * e)
        tz = (c & -c).bit_length() - 1
        lvl = e - tz
        p = (c >> tz) >> 1
        return lvl_off(lvl) + p * stride(lvl) + tri_ix(2 * (Q0 - lvl), 2 * tz, 2 * tz)

    return stride, lvl_off, node_off


def wf(addrs, width):
    """wavefronts of one warp access; addrs in units of `width` bytes, None = inactive lane.
    8- and 16-byte accesses are served per 16- / 8-lane phase (128 bytes each): per phase, the
    max over the 128/width bank slots of the distinct addresses in the slot"""
    slots = 128 // width
    ph = 32 * width // 128 if width > 4 else 1
    n = 32 // ph
    tot = ideal = 0
    for p in range(ph):
        per = collections.defaultdict(set)
        for a in addrs[p * n:(p + 1) * n]:
            if a is not None:
                per[a % slots].add(a)
        if per:
            tot += max(len(v) for v in per.values())
            ideal += 1
    return tot, ideal


def ij_of(D):
    out = []
    for i in range(D):
        for j in range(i, D):
            out.append((i, j))
    return out


def pair_stride(e, G):
    m = 2 * (Q0 - e + 1)
    if G >= 8:
        return m + 1
    st = m
    while st % 8 != G % 8:
        st += 1
    return st


def cost(pads, adds, maps, pstr=None, detail=False):
    stride, lvl_off, node_off = layout(pads, adds)
    tot = ideal = 0
    rows = []
    for e in range(1, FAN + 1):
        E = 1 << (e - 1)
        G = 32 // E
        m = 2 * (Q0 - e + 1)
        D = m - 2
        tn = tri(D)
        ij = ij_of(D)
        S2 = m + pstr[e - 1] if pstr else pair_stride(e, G)
        lanes = []
        for lane in range(32):
            if maps[e - 1] == 0:
                x, g = lane // G, lane % G
            else:
                x, g = lane % E, lane // E
            lanes.append((x, g))
        acc = []
        # pivot loads P[0], P[1], P[m]
        for off in (0, 1, m):
            acc.append((wf([node_off(e - 1, x) + off for x, g in lanes], 8), 1))
        NVS = -(-(m - 2) // G)
        for s in range(NVS):
            for base in (2, m + 1):
                acc.append((wf([node_off(e - 1, x) + base + g + s * G for x, g in lanes], 8), 1))
            acc.append((wf([(x * S2 + 2 + g + s * G) if g + s * G < m - 2 else None for x, g in lanes], 16), 1))
        NS = -(-tn // G)
        for s in range(NS):
            ks = [(x, g + s * G) for x, g in lanes]
            act = [(x, k) if k < tn else None for x, k in ks]
            acc.append((wf([None if a is None else node_off(e - 1, a[0]) + 2 * m - 1 + a[1] for a in act], 8), 1))
            acc.append((wf([None if a is None else lvl_off(e) + a[0] * stride(e) + a[1] for a in act], 8), 1))
            acc.append((wf([None if a is None else a[0] * S2 + 2 + ij[a[1]][0] for a in act], 16), 1))
            acc.append((wf([None if a is None else a[0] * S2 + 2 + ij[a[1]][1] for a in act], 16), 1))
        lt = sum(a[0][0] * a[1] for a in acc)
        li = sum(a[0][1] * a[1] for a in acc)
        rows.append((e, lt, li))
        tot += lt
        ideal += li
    # lane subtrees: ~91 loads per lane tree at compile-time offsets from node (5, lane)
    b = [node_off(5, c) for c in range(32)]
    lw = wf(b, 8)
    tot += 91 * lw[0]
    ideal += 91 * lw[1]
    rows.append(("lanes", 91 * lw[0], 91 * lw[1]))
    if detail:
        return tot, ideal, rows
    return tot, ideal


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    cur_pads, cur_adds = [0, 0, 1, 2, 8], [1, 0, 3, 0, 0]  # round-2 layout (lane-subtree search)
    for maps in ([0] * 5, [1] * 5):
        t, i, rows = cost(cur_pads, cur_adds, maps, detail=True)
        print("current layout, maps", maps, "wavefronts/leaf", t, "ideal", i, rows)
    stride, lvl_off, _ = layout([0] * 5, [0] * 5)
    base_end = lvl_off(FAN + 1)
    rng = random.Random(7)
    best = None

    def obj(p, a, mp, ps):
        t, _ = cost(p, a, mp, ps)
        _, lo, _ = layout(p, a)
        return (t, lo(FAN + 1) - base_end)

    for r in range(iters):
        p = [rng.randrange(16) for _ in range(5)]
        a = [rng.randrange(8) for _ in range(5)]
        mp = [rng.randrange(2) for _ in range(5)]
        ps = [1 + rng.randrange(8) for _ in range(5)]
        cur = obj(p, a, mp, ps)
        improved = True
        while improved:
            improved = False
            for i in range(5):
                for v in range(16):
                    q = p[:]
                    q[i] = v
                    o = obj(q, a, mp, ps)
                    if o < cur:
                        cur, p, improved = o, q, True
                for v in range(8):
                    q = a[:]
                    q[i] = v
                    o = obj(p, q, mp, ps)
                    if o < cur:
                        cur, a, improved = o, q, True
                for v in range(1, 9):
                    q = ps[:]
                    q[i] = v
                    o = obj(p, a, mp, q)
                    if o < cur:
                        cur, ps, improved = o, q, True
                q = mp[:]
                q[i] ^= 1
                o = obj(p, a, q, ps)
                if o < cur:
                    cur, mp, improved = o, q, True
        if best is None or cur < best[0]:
            best = (cur, p, a, mp, ps)
            print(r, best, flush=True)
    t, i, rows = cost(best[1], best[2], best[3], best[4], detail=True)
    print("best", best, "ideal", i, rows)


if __name__ == "__main__":
    main()
