"""The bench.py JSON line contract (driver-facing): the committed round line carries every
required key, and (on a GPU) a short bench run prints one well-formed line."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks")


def _check_line(d: dict, cpu: bool):
    for k in REQUIRED:
        assert k in d, k
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] < 1 and abs(r["achieved"] / r["peak"] - r["frac"]) < 1e-9
    if cpu:
        c = d["cpu_baseline"]
        assert c["value"] > 0 and c["cores"] >= 1 and c["kind"] in ("reference", "port") and c["sample"]


def test_committed_bench_line():
    d = json.load(open(os.path.join(ROOT, "profiles", "r01_bench.json")))
    _check_line(d, cpu=True)
    assert d["config"]["workload"] == "cfg4-n32-dd" and d["n_gpus"] == 1
    ref = json.load(open(os.path.join(ROOT, "profiles", "r01_bench_reference.json")))
    assert ref["impl"] == "reference" and ref["metric"] == d["metric"] and ref["unit"] == d["unit"]
    assert ref["e2e"]["h2d_bytes_per_step"] == 0 and ref["cpu_baseline"]["value"] == ref["value"]


def test_committed_round2_bench_lines():
    d = json.load(open(os.path.join(ROOT, "profiles", "r02_bench.json")))
    _check_line(d, cpu=True)
    assert d["config"]["workload"] == "cfg4-n32-dd" and d["n_gpus"] == 1 and d["steps"] == 20 and d["warmup"] == 5
    assert d["cpu_baseline"]["unit"] == d["unit"] and d["clocks"]["reasons"] == []
    ref = json.load(open(os.path.join(ROOT, "profiles", "r02_bench_reference.json")))
    assert ref["impl"] == "reference" and ref["metric"] == d["metric"] and ref["config"]["workload"] == "cfg4-n32-dd"
    for w in ("cfg4-n32-qd", "cfg5-n40-dd", "cfg3-batch-fp64", "cfg3-batch-dd"):
        _check_line(json.load(open(os.path.join(ROOT, "profiles", f"r02_bench_{w}.json"))), cpu=True)


@pytest.mark.gpu
def test_bench_runs_and_prints_one_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "3",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    _check_line(d, cpu=False)
    assert d["result"]["value"] == pytest.approx(7.40836601865894e-11, rel=1e-12)


def test_reference_arm_runs_on_host():
    # bench.py --impl reference times the reference's own fixed-point engine (oracle/_ref, or
    # the C restatement when the reference was not built) on the host cores: no GPU involved
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1", "--cpu-sample-seconds", "1"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "subset-terms/s"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["cpu_baseline"]["unit"] == d["unit"]
