"""CPU: SASS-count regression on the committed DD/QD inner loops (north_star item 3).

profiles/sass/ holds the cuobjdump -sass listings of the arithmetic primitives (the probes of
tools/probes/prims.cu, compiled with the engine's flags) and of subtree_kernel<dd>, plus the
FP64 instruction counts of every probe and every engine kernel (tools/sass_commit.py).  These
tests recompile / disassemble and compare:
  - the probes' counts == the committed listings == profiles/flops_model.json's SASS counts
    (the roofline's algorithmic flops/term are built from these primitives);
  - the built libtor_b200.so's per-kernel counts == profiles/sass/counts.json whenever the
    kernel sources are the ones the counts were committed from.
"""
from __future__ import annotations

import json
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = pytest.mark.skipif(shutil.which("nvcc") is None or shutil.which("cuobjdump") is None,
                                reason="needs nvcc / cuobjdump")

import sass_commit as S  # noqa: E402

COUNTS = json.load(open(os.path.join(ROOT, "profiles", "sass", "counts.json")))
KEY_PRIMS = ("rank2_dd", "pivot_dd", "leaf_dd", "vec_dd", "rank2_qd", "pivot_qd", "leaf_qd", "vec_qd")


@pytest.fixture(scope="module")
def probes():
    return S.split_functions(S.probe_sass())


def test_committed_listings_exist_for_the_inner_loops():
    for p in KEY_PRIMS:
        path = os.path.join(ROOT, "profiles", "sass", f"prims_{p}.sass")
        assert os.path.exists(path), path
        body = open(path).read().split("\n")
        assert S.count(body) == COUNTS["probes"][p]
    dd = open(os.path.join(ROOT, "profiles", "sass", "subtree_kernel_dd.sass")).read().split("\n")
    assert S.count(dd) == COUNTS["engine"]["subtree_kernel<dd>"]


def test_probe_counts_match_committed_sass(probes):
    got = {k: S.count(v) for k, v in probes.items()}
    for p in KEY_PRIMS:
        assert got[p] == COUNTS["probes"][p], p
    # the DD rank-2 entry update of the biased grid: 8 DFMA + 4 DADD
    assert (got["rank2_dd"]["DFMA"], got["rank2_dd"]["DADD"], got["rank2_dd"]["DMUL"]) == (8, 4, 0)


def test_flops_model_uses_these_primitives(probes):
    fm = json.load(open(os.path.join(ROOT, "profiles", "flops_model.json")))
    got = {k: S.count(v) for k, v in probes.items()}
    for name, c in fm["primitives_sass_probe"].items():
        assert {k: got[name][k] for k in S.OPS} == c, name


def test_engine_kernels_match_committed_counts():
    if S.sources_sha() != COUNTS["sources_sha256"]:
        pytest.fail("kernel sources changed since profiles/sass was committed: run tools/sass_commit.py")
    eng = {S.short(k): S.count(v) for k, v in S.split_functions(S.engine_sass()).items()}
    for k, c in COUNTS["engine"].items():
        assert eng.get(k) == c, k
