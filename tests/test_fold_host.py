"""CPU: tor_fold_partials (host code, no device) -- the fold of shard / class partials along
the engine's fixed tree, its input checks, and the FixedValue limbs it reports.

The reference's fan-out folds per-worker partials exactly (run_engine, torontonian.cpp:112-147,
limb-identical for any worker count, tests/test_torontonian.cpp:120-155).  Here a fold is
bit-identical to one device when every partial spans an aligned power-of-two class block: the
fold of blocks equals the fold of the classes inside them.
"""
from __future__ import annotations

import random

import pytest

import paper_2009_01177_b200 as T
from paper_2009_01177_b200 import api
from paper_2009_01177_b200 import workloads as W

M = W.load_config_instance(2)  # n = 20
N = M.n_modes


def part(mode, k, lo, hi, words, sum_abs=1.0):
    return dict(mode=mode, class_bits=k, class_lo=lo, class_hi=hi, words=tuple(words), sum_abs=sum_abs,
                term_count=(hi - lo) << (N - k))


def rnd_words(rng, nw):
    x = rng.uniform(-1, 1) * 2.0 ** rng.randint(-40, 0)
    w = [x]
    for _ in range(nw - 1):
        w.append(w[-1] * rng.uniform(-1, 1) * 2.0 ** -53)
    return w + [0.0] * (4 - nw)


@pytest.mark.parametrize("mode,nw", [(api.PREC_DD, 2), (api.PREC_QD, 4)])
def test_fold_of_blocks_equals_fold_of_classes(mode, nw):
    rng = random.Random(7 + nw)
    k = 3
    leaves = [part(mode, k, c, c + 1, rnd_words(rng, nw), rng.uniform(1, 2)) for c in range(8)]
    whole = T.fold_partials(leaves, M)

    def sub(lo, hi):  # the tree's subtree fold over classes [lo, hi) via a smaller class grid
        w = hi - lo
        kk = w.bit_length() - 1
        ps = [dict(p, class_bits=kk, class_lo=i, class_hi=i + 1, term_count=1 << (N - kk))
              for i, p in enumerate(leaves[lo:hi])]
        r = T.fold_partials(ps, M)
        return part(mode, k, lo, hi, r["words"] + (0.0,) * (4 - len(r["words"])), r["sum_abs_terms"])

    for cover in ([(0, 4), (4, 8)], [(0, 2), (2, 3), (3, 4), (4, 8)], [(0, 1), (1, 2), (2, 4), (4, 6), (6, 7), (7, 8)]):
        blocks = [sub(lo, hi) if hi - lo > 1 else leaves[lo] for lo, hi in cover]
        r = T.fold_partials(blocks, M)
        assert r["words"] == whole["words"], cover
        assert r["sum_abs_terms"] == whole["sum_abs_terms"]
    # the reported limbs are the exact re-quantisation of the folded words
    assert whole["raw_limbs"] == api.raw_limbs(whole["words"], whole["width_bits"], whole["config"]["frac_bits"])


def test_fold_rejects_bad_partial_sets():
    rng = random.Random(3)
    leaves = [part(api.PREC_DD, 2, c, c + 1, rnd_words(rng, 2)) for c in range(4)]
    T.fold_partials(leaves, M)
    bad_sets = {
        "missing last": leaves[:3],
        "missing first": leaves[1:],
        "gap": [leaves[0], leaves[2], leaves[3]],
        "mixed modes": [leaves[0], dict(leaves[1], mode=api.PREC_QD), leaves[2], leaves[3]],
        "mixed class bits": [leaves[0], dict(leaves[1], class_bits=3), leaves[2], leaves[3]],
        "unaligned block": [leaves[0], part(api.PREC_DD, 2, 1, 3, rnd_words(rng, 2)), leaves[3]],
        "non-power-of-two block": [part(api.PREC_DD, 2, 0, 3, rnd_words(rng, 2)), leaves[3]],
        "term count": [leaves[0], dict(leaves[1], term_count=5), leaves[2], leaves[3]],
        "auto mode": [dict(p, mode=api.PREC_AUTO) for p in leaves],
        "fixed mode": [dict(p, mode=api.PREC_FIXED128) for p in leaves],
    }
    for why, ps in bad_sets.items():
        with pytest.raises(T.InvalidArgument):
            T.fold_partials(ps, M)
            pytest.fail(why)


@pytest.mark.parametrize("seed", range(20))
def test_requantised_limbs_exact(seed):
    """C requantise (round(sum words * 2^f), ties up, two's complement) == exact Python."""
    rng = random.Random(seed)
    for mode, nw in ((api.PREC_DD, 2), (api.PREC_QD, 4)):
        w = rnd_words(rng, nw)
        if seed % 3 == 0:
            w[0] = -w[0]
        r = T.fold_partials([part(mode, 0, 0, 1, w)], M)
        assert r["words"][:nw] == tuple(w[:nw])
        assert r["raw_limbs"] == api.raw_limbs(r["words"], r["width_bits"], r["config"]["frac_bits"])
