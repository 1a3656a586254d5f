"""CPU, world_size 2 and 4 over gloo: the multi-rank path of bench.py / INTEGRATION.md.

Each rank owns the power-of-two aligned prefix classes [rank, rank+1) of the top
log2(world) mask bits (paper_2009_01177_b200.subsets.prefix_classes), computes its
shard partial, all-gathers the 10-double partial records, and folds them with the
engine's host-side fixed-order fold (tor_fold_partials).  On CPU the shard partials
come from the oracle (exact fixed point, converted to DD words); the plumbing and
the fold are the product code.  The result must be identical on every rank and for
every world size, and equal the reference's full value.
"""
from __future__ import annotations

import os
import socket
from fractions import Fraction

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests._util import fixed_value


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dd_words(x: Fraction):
    hi = float(x)
    lo = float(x - Fraction(hi))
    return (hi, lo, 0.0, 0.0)


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2009_01177_b200 as T
        from oracle import port as P
        from paper_2009_01177_b200 import api
        from paper_2009_01177_b200 import workloads as W
        m = W.load_config_instance(1)
        k, lo, hi = T.prefix_classes(m.n_modes, rank, world)
        f = T.force_width(m, 128)["frac_bits"]
        tot, per, sabs = P.slice(m, 128, f, k, lo, hi, threads=2)
        part = dict(mode=api.PREC_DD, class_bits=k, class_lo=lo, class_hi=hi,
                    words=_dd_words(Fraction(tot, 1 << f)), sum_abs=sum(sabs), term_count=(hi - lo) << (16 - k))
        buf = torch.tensor(api.partial_to_array(part), dtype=torch.float64)
        gathered = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(gathered, buf)
        parts = [api.array_to_partial(g.numpy()) for g in gathered]
        r = T.fold_partials(parts, m)
        out_q.put((rank, tuple(r["words"]), r["term_count"], r["sum_abs_terms"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_shards_fold_identically(world, golden):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    words = {r[1] for r in res}
    assert len(words) == 1, "every rank must fold to the same words"
    w, terms, sabs = res[0][1], res[0][2], res[0][3]
    assert terms == 1 << 16
    g = golden["cfg1"]["fixed128"]
    want = fixed_value(g["raw"], g["frac_bits"])
    got = sum((Fraction(x) for x in w), Fraction(0))
    # exact shard sums; the fold adds < 2^-100 sum|t|
    assert abs(float(got - want)) <= 2.0 ** -100 * sabs


def _bench_worker(rank, world, port, out_q):
    """bench.py's own multi-rank code (split_classes + gather_fold) with stub class partials:
    exact fixed-point class sums from the oracle instead of the GPU."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench
        import paper_2009_01177_b200 as T
        from oracle import port as P
        from paper_2009_01177_b200 import api
        from paper_2009_01177_b200 import workloads as W
        m = W.load_config_instance(1)
        lo, hi = bench.split_classes(rank, world)
        f = T.force_width(m, 128)["frac_bits"]
        k = bench.KBITS
        tot, per, sabs = P.slice(m, 128, f, k, lo, hi, threads=2)
        mine = [dict(mode=api.PREC_DD, class_bits=k, class_lo=c, class_hi=c + 1,
                     words=_dd_words(Fraction(v, 1 << f)), sum_abs=sa, term_count=1 << (16 - k))
                for c, v, sa in zip(range(lo, hi), per, sabs)]
        r = bench.gather_fold(mine, world, m, dist)
        out_q.put((rank, tuple(r["words"]), r["term_count"], r["sum_abs_terms"], hi - lo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 6])
def test_bench_multirank_plumbing_any_world(world, golden):
    """Any world size (not only powers of two): every rank folds the same 64 class partials."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len({r[1] for r in res}) == 1
    assert sum(r[4] for r in res) == 64 and max(r[4] for r in res) - min(r[4] for r in res) <= 1
    w, terms, sabs = res[0][1], res[0][2], res[0][3]
    assert terms == 1 << 16
    g = golden["cfg1"]["fixed128"]
    got = sum((Fraction(x) for x in w), Fraction(0))
    assert abs(float(got - fixed_value(g["raw"], g["frac_bits"]))) <= 2.0 ** -100 * sabs


def test_bench_refuses_more_gpus_than_visible():
    """--gpus N is honoured or refused: without N devices bench.py exits non-zero."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "3", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert out.returncode != 0
    assert "requested" in out.stdout
