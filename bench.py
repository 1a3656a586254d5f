#!/usr/bin/env python3
"""Benchmark of the B200 Torontonian engine (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N --steps K --warmup W] [--impl engine|reference] [--workload ...]

Headline (BASELINE.json metric): Torontonian subset-terms/sec, n=32, double-double, on
config 4's input (the headline row in DD on config 4's input).  One step =
one full Torontonian (2^32 subset-terms) evaluated on the GPU.  With --gpus N > 1 (run under
torchrun, or self-launched through torch.distributed.run when WORLD_SIZE is unset) rank r
evaluates the top-level prefix classes [64r/N, 64(r+1)/N) of the top 6 mask bits (strong
scaling: total work fixed; any N <= 64), the per-class partials are all-gathered over NCCL
and every rank folds all 64 along the engine's fixed tree (bit-identical for any N).

value  : terms/s with the exact R resident in HBM (tor_plan_execute), device-timed with
         CUDA events, max over ranks.
e2e    : same metric through the public C ABI call tor_torontonian / tor_torontonian_shard
         with host buffers (host prep + H2D + device + D2H inside the timed region).
--impl reference : the reference's own CPU engine (oracle/_ref = unmodified torfp
         sources built by oracle/Makefile; the C restatement oracle/liboracle.so if that is
         missing) on the box's host cores, bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Torontonian subset-terms/sec (n=32, double-double)"
UNIT = "subset-terms/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--workload", default="cfg4-n32-dd",
                    choices=["cfg4-n32-dd", "cfg4-n32-qd", "cfg2-n20-dd", "cfg1-n16-fp64", "cfg5-n40-dd",
                             "cfg3-batch-fp64", "cfg3-batch-dd"])
    ap.add_argument("--cpu-sample-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# ------------------------------------------------------------- multi-rank ----
KBITS = 6  # top-level prefix classes split across ranks (tor_torontonian_classes)


def split_classes(rank: int, world: int) -> tuple[int, int]:
    """Contiguous class range of `rank` (sizes differ by at most one class)."""
    n = 1 << KBITS
    if not 1 <= world <= n or not 0 <= rank < world:
        raise SystemExit(f"bench.py: world size must be in [1, {n}] (got {world})")
    return n * rank // world, n * (rank + 1) // world


def gather_fold(parts: list[dict], world: int, m, dist, device=None) -> dict:
    """All-gather this rank's per-class partials (10 doubles each, padded to the largest
    rank's count) and fold all 2^KBITS classes along the fixed tree (tor_fold_partials,
    host code): every rank returns the same words."""
    import torch
    from paper_2009_01177_b200 import api
    import paper_2009_01177_b200 as T
    width = (1 << KBITS) // world + 1
    buf = torch.full((width, 10), -1.0, dtype=torch.float64)
    for i, p in enumerate(parts):
        buf[i] = torch.from_numpy(api.partial_to_array(p))
    if device is not None:
        buf = buf.to(f"cuda:{device}")
    allb = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(allb, buf)
    got = []
    for b in allb:
        for row in b.cpu().numpy():
            if row[3] >= 0:  # class_hi of a real record (padding rows are -1)
                got.append(api.array_to_partial(row))
    return T.fold_partials(sorted(got, key=lambda p: p["class_lo"]), m)


def self_launch(args) -> int:
    """--gpus N > 1 without torchrun: relaunch this script as N NCCL ranks (the driver's own
    launch form); refuse (exit 2) when the node has fewer than N GPUs."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} requested but {have} CUDA device(s) visible"}), flush=True)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


WORKLOADS = {
    "cfg4-n32-dd": (4, "128", "dd"),
    "cfg4-n32-qd": (4, "256", "qd"),
    "cfg2-n20-dd": (2, "128", "dd"),
    "cfg1-n16-fp64": (1, "fp64", "fp64"),
    "cfg5-n40-dd": (5, "128", "dd"),
    "cfg3-batch-fp64": (3, "fp64", "fp64"),
    "cfg3-batch-dd": (3, "128", "dd"),
}
BATCH = 4096  # BASELINE config 3: 4096 Torontonians, n = 16 each
DATA = "synthetic (seeded pure Gaussian state, SURVEY 8(d) recipe; committed input tests/golden/cfg{}.gbsa.txt)"


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """Samples SM clock + throttle reasons during the timed region (NVML)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------- fp64 peak ----
def fp64_peak_tflops(device: int):
    """Live DFMA microbenchmark (tools/fp64_peak), the FP64 roofline denominator
    (MEASURED_PEAKS.json has no FP64 entry)."""
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    why = "tools/fp64_peak missing"
    if os.path.exists(exe):
        try:
            out = subprocess.run([exe], capture_output=True, text=True, timeout=60,
                                 env=dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "")))
            d = json.loads(out.stdout.strip().splitlines()[-1])
            return d["dfma_tflops"], ("measured: tools/fp64_peak DFMA microbenchmark (best of 8-32 independent "
                                      "chains x 4/8 CTAs per SM, this box)")
        except Exception as e:  # pragma: no cover
            why = f"fp64_peak failed: {e}"
    # fallback: the committed measurement of the same microbenchmark on this pool's B200s
    rec = os.path.join(ROOT, "profiles", "r02_fp64_peak.json")
    if os.path.exists(rec):
        return json.load(open(rec))["dfma_tflops"], f"recorded: profiles/r02_fp64_peak.json ({why})"
    return None, why


# -------------------------------------------------------------- baseline ----
def ref_sample(m, precision: str, seconds: float):
    """Reference CPU engine timed on a bounded sample (all host threads)."""
    from oracle import ref
    threads = os.cpu_count() or 1
    n = m.n_modes
    if ref.available() and precision == "fp64" and n <= 20:
        # the reference's fp64 path (torontonian_reference, torontonian.cpp:179-200) is a
        # single-threaded call: the whole instance on every host thread concurrently
        return ref_batch_sample([m] * max(threads, 1) * 64, "fp64", seconds)
    if ref.available():
        # torontonian_partial over partition(n, rank, nproc) slices: each rank's share keeps
        # the popcount mix of the full sum; calibrate the sample to ~`seconds`
        width = {"128": "128", "dd": "128", "256": "256", "qd": "256"}.get(precision, "128")
        nproc = 1 << max(5, min(30, n - 8))  # >= 256 subset-terms per partition rank
        done, secs = ref.partial_sample(m, width, nproc, 0, threads, threads)
        rate = done / max(secs, 1e-9)
        target = max(threads, int(rate * seconds))
        nranks = min(threads * max(1, round(target / max(done, 1))), nproc - threads)
        done, secs = ref.partial_sample(m, width, nproc, threads, nranks, threads)
        return dict(value=done / secs, unit=UNIT, cores=threads, kind="reference",
                    sample=f"torfp torontonian_partial<{'2' if width == '128' else '4'}> (fixed-{width}) over "
                           f"{nranks} of {nproc} partition ranks of n={n}: {done} subset-terms in {secs:.2f} s "
                           f"on {threads} threads")
    from oracle import port
    done, secs = port.partial_sample(m, 128 if precision in ("128", "dd") else 256, seconds, threads)
    return dict(value=done / secs, unit=UNIT, cores=threads, kind="port",
                sample=f"oracle/tor_oracle.c fixed-point restatement: {done} subset-terms in {secs:.2f} s")


def ref_batch_sample(ms, precision: str, seconds: float):
    """Reference CPU engine on a bounded sample of the config-3 items: fp64 = the reference's
    fp64 path torontonian_reference (torontonian.cpp:179, single-threaded per call: items run
    concurrently on all host threads); 128 = torontonian(a, Bits128, workers = host cores) item
    after item.  Returns terms/s over the sample."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import ref
    threads = os.cpu_count() or 1
    n = ms[0].n_modes
    if not ref.available():
        from oracle import port
        done, secs = port.partial_sample(ms[0], 128, seconds, threads)
        return dict(value=done / secs, unit=UNIT, cores=threads, kind="port",
                    sample=f"oracle/tor_oracle.c fixed-point restatement: {done} subset-terms in {secs:.2f} s")
    done, t0, k = 0, time.perf_counter(), 0
    if precision == "fp64":
        with ThreadPoolExecutor(threads) as ex:
            while time.perf_counter() - t0 < seconds and k < len(ms):
                list(ex.map(ref.reference_timed, ms[k:k + threads]))
                k += len(ms[k:k + threads])
        what = f"torfp torontonian_reference (fp64) on {k} of the {len(ms)} config-3 items, {threads} concurrent calls"
    else:
        while time.perf_counter() - t0 < seconds and k < len(ms):
            ref.torontonian(ms[k], "128", threads)
            k += 1
        what = f"torfp torontonian(Bits128, workers={threads}) on {k} of the {len(ms)} config-3 items"
    secs = time.perf_counter() - t0
    return dict(value=k * (1 << n) / secs, unit=UNIT, cores=threads, kind="reference",
                sample=f"{what}: {k * (1 << n)} subset-terms in {secs:.2f} s")


def batch_main(args, cfg, prec, dtype):
    """Config 3: 4096 Torontonians (n = 16) per step through tor_torontonian_batch.
    value: terms/s of the device pipeline (CUDA events, inputs already uploaded: the engine's
    device_ms); e2e: the C-ABI call on host arrays (validation, exact R, host->device copy,
    device pipeline, results) timed on the host."""
    import paper_2009_01177_b200 as T
    from paper_2009_01177_b200 import workloads as W
    ms = W.load_cfg3_batch(BATCH)
    n = ms[0].n_modes
    terms = BATCH * (1 << n)
    if args.impl == "reference":
        vals = []
        for s in range(args.warmup + args.steps):
            r = ref_batch_sample(ms, prec, max(2.0, args.cpu_sample_seconds / 3))
            if s >= args.warmup:
                vals.append(r["value"])
        v = statistics.median(vals)
        print(json.dumps({"metric": f"Torontonian subset-terms/sec ({args.workload})", "value": v, "unit": UNIT,
                          "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": terms / v * 1e3, "higher_is_better": True,
                          "ms_per_step_note": "derived: terms per step / value (bounded sample per step)",
                          "scaling": "strong", "vs_baseline": None, "dtype": "fixed-128" if dtype == "dd" else dtype,
                          "data": DATA.format("3_state"), "impl": "reference",
                          "config": {"workload": args.workload, "n": n, "instances": BATCH, "precision": prec},
                          "cpu_baseline": dict(r, value=v),
                          "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    import torch
    torch.cuda.set_device(0)
    batch = T.api.BatchInputs(ms)
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda:0")
    for _ in range(args.warmup):
        T.api.torontonian_batch_raw(batch, prec)
    dev_ms, kern_ms, e2e_ms = [], [], []
    with ClockSampler(0) as clk:
        t_all = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = T.api.torontonian_batch_raw(batch, prec)
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
            dev_ms.append(float(r["device_ms"][0]))
            kern_ms.append(float(r["kernel_ms"][0]))
        wall = time.perf_counter() - t_all
    step_ms, kstep = statistics.median(dev_ms), statistics.median(kern_ms)
    peak, peak_src = fp64_peak_tflops(0)
    fm = json.load(open(os.path.join(ROOT, "profiles", "flops_model.json")))["per_term"][dtype][str(n)]
    achieved = terms * fm["flops"] / (kstep * 1e-3) / 1e12
    words = {"fp64": 1, "dd": 2}[dtype]
    line = {"metric": f"Torontonian subset-terms/sec ({args.workload})", "value": terms / (step_ms * 1e-3),
            "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype,
            "data": DATA.format("3_state"),
            "config": {"workload": args.workload, "n": n, "instances": BATCH, "precision": prec,
                       "terms_per_step": terms, "l2": "flushed between steps (256 MiB write)"},
            "e2e": {"value": terms / (statistics.median(e2e_ms) * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": BATCH * (2 * n) * (2 * n + 1) // 2 * words * 8,
                    "d2h_bytes_per_step": BATCH * 40 + 8, "ms_per_step": statistics.median(e2e_ms),
                    "over_device": statistics.median(e2e_ms) / step_ms,
                    "path": "tor_torontonian_batch on host arrays (ctypes): validation, exact R into pinned "
                            "staging, host->device copy, device pipeline, results"},
            "gpu_launches": int(r["kernel_launches"][0]) * args.steps, "kernel_ms_per_step": kstep,
            "result": {"item0": float(r["value"][0]), "sum_abs_item0": float(r["sum_abs_terms"][0])},
            "clocks": clk.summary(), "wall_s_timed": wall,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": None, "kernel": "subtree_kernel",
                         "flops_per_term": fm["flops"], "peak_source": peak_src}}
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = ref_batch_sample(ms, prec, args.cpu_sample_seconds)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ main ----
def main():
    args = parse()
    cfg, prec, dtype = WORKLOADS[args.workload]
    if args.workload.startswith("cfg3-batch"):
        if int(os.environ.get("RANK", "0")) == 0:
            batch_main(args, cfg, prec, dtype)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "engine":
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "engine" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    from paper_2009_01177_b200 import workloads as W
    m = W.load_config_instance(cfg)
    n = m.n_modes
    terms_total = 1 << n

    if args.impl == "reference":
        if rank != 0:
            return
        times, vals = [], []
        for s in range(args.warmup + args.steps):
            r = ref_sample(m, prec, max(2.0, args.cpu_sample_seconds / 3))
            if s >= args.warmup:
                vals.append(r["value"])
        v = statistics.median(vals)
        line = {"metric": METRIC if args.workload == "cfg4-n32-dd" else f"Torontonian subset-terms/sec ({args.workload})",
                "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": terms_total / v * 1e3, "higher_is_better": True,
                "ms_per_step_note": "derived, not timed: 2^n / value -- each step times a bounded sample "
                                    "(cpu_baseline.sample) of the same Torontonian, the full sum would take "
                                    f"{terms_total / v / 3600:.0f} h on these cores",
                "scaling": "strong", "vs_baseline": None, "dtype": "fixed-128" if dtype == "dd" else dtype,
                "data": DATA.format(cfg), "impl": "reference",
                "config": {"workload": args.workload, "n": n, "precision": prec},
                "cpu_baseline": dict(r, value=v),
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    import paper_2009_01177_b200 as T

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", init_method="env://")
    device = local if world > 1 else 0
    torch.cuda.set_device(device)
    # resident-input plan for this rank's share of the top-level prefix classes
    if world > 1:
        k, (clo, chi) = KBITS, split_classes(rank, world)
    else:
        k, clo, chi = 0, 0, 1
    plan = T.api.Plan(m, prec, k, clo, chi, device=device)
    flush = torch.empty(64 << 20, dtype=torch.int32, device=f"cuda:{device}")  # 256 MiB > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        plan.execute()
    # ---- value: device-resident inputs, device time (CUDA events inside the plan)
    dev_ms, kern_ms, parts, launches = [], [], None, 0
    peak, peak_src = (fp64_peak_tflops(device) if rank == 0 else (None, None))
    with ClockSampler(device) as clk:
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            flush.zero_()  # L2 flush between steps (outside the plan's event window)
            r = plan.execute()
            dev_ms.append(r["device_ms"])
            kern_ms.append(r["kernel_ms"])
            launches = r["kernel_launches"]
            parts = r
        barrier()
        wall_steps = time.perf_counter() - t0
    step_ms = sum(dev_ms) / len(dev_ms)
    kstep_ms = sum(kern_ms) / len(kern_ms)
    if world > 1:
        t = torch.tensor([step_ms, kstep_ms], device=f"cuda:{device}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms, kstep_ms = float(t[0]), float(t[1])
    value = terms_total / (step_ms * 1e-3)

    # ---- e2e: public API with host buffers, all ranks, fold over NCCL
    e2e_ms = []
    result = None
    for s in range(args.warmup + args.steps):
        barrier()
        t0 = time.perf_counter()
        if world > 1:
            mine = T.torontonian_classes(m, prec, KBITS, clo, chi, device=device)
            result = gather_fold(mine, world, m, dist, device)
        else:
            result = T.torontonian(m, prec)
        barrier()
        dt = (time.perf_counter() - t0) * 1e3
        if world > 1:
            tt = torch.tensor([dt], device=f"cuda:{device}", dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt[0])
        if s >= args.warmup:
            e2e_ms.append(dt)
    e2e_step = statistics.median(e2e_ms)
    # bytes moved per step, all ranks: each rank uploads the exact R (the single-device
    # call reports its own counts) and reads back its class partials (5 doubles each + the
    # error word); with N > 1 each rank also uploads its padded partial records for the
    # all-gather and reads the N gathered blocks back
    words = {"fp64": 1, "dd": 2, "qd": 4}[dtype]
    r_bytes = (2 * n) * (2 * n + 1) // 2 * words * 8
    if world == 1:
        h2d_step, d2h_step = int(result.get("h2d_bytes", r_bytes)), int(result.get("d2h_bytes", 48))
    else:
        rec = ((1 << KBITS) // world + 1) * 80
        h2d_step = world * (r_bytes + rec)
        d2h_step = (1 << KBITS) * 40 + world * 8 + world * world * rec

    if rank == 0:
        def _load(name):
            path = os.path.join(ROOT, "profiles", name)
            return json.load(open(path)) if os.path.exists(path) else {}
        fmodel = _load("flops_model.json").get("per_term", {}).get(dtype, {}).get(str(n), {})
        sass = _load("sass_counts.json")
        fpt = fmodel.get("flops")          # algorithmic flops / term (SASS-pinned primitive model)
        ipt = fmodel.get("fp64_instr")
        roof = None
        if fpt and peak:
            # the most loaded rank bounds the max-over-ranks kernel time
            terms_rank = terms_total * (-(-(1 << KBITS) // world) if world > 1 else 1) / ((1 << KBITS) if world > 1 else 1)
            achieved = terms_rank * fpt / (kstep_ms * 1e-3) / 1e12
            roof = {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": sass.get("dram_bytes_per_launch", {}).get(dtype),
                    "kernel": "subtree_kernel", "flops_per_term": fpt,
                    "flops_per_term_source": "profiles/flops_model.json: Schur-tree node counts x SASS-pinned "
                                             "primitive costs (tools/flops_model.py), useful work only",
                    "kappa": fmodel.get("kappa"), "rho": fmodel.get("rho_leaf_bundle_flops"),
                    "peak_source": peak_src}
            # nominal 64 DFMA/clk/SM x SMs x max clock x 2 flops (the microbenchmark sustains
            # ~58.5/clk/SM at any chain count: profiles/r02_fp64_peak.json)
            import torch
            sms = torch.cuda.get_device_properties(device).multi_processor_count
            mhz = clk.summary().get("sm_max_mhz") or 1965
            roof["peak_nominal"] = 2 * 64 * sms * mhz * 1e6 / 1e12
            roof["frac_nominal"] = achieved / roof["peak_nominal"]
            if ipt:
                # FP64 pipe issue utilisation: DD arithmetic is DADD-heavy, so the flop
                # fraction caps well below 1 even at a saturated pipe (peak = 2 flops/instr)
                roof["fp64_instr_per_term"] = ipt
                roof["fp64_pipe_frac"] = terms_rank * ipt / (kstep_ms * 1e-3) / (peak * 1e12 / 2)
            ex = sass.get("flops_per_term", {}).get(dtype)
            if ex:
                # cross-check: ncu executed (includes lanes that compute warp-uniform pivots
                # redundantly and padding items)
                roof["executed_flops_per_term_ncu"] = ex
                roof["executed_over_algorithmic"] = ex / fpt
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                cpu = ref_sample(m, prec, args.cpu_sample_seconds)
            except Exception as e:  # pragma: no cover
                cpu = {"error": str(e)}
        line = {
            "metric": METRIC if args.workload == "cfg4-n32-dd" else f"Torontonian subset-terms/sec ({args.workload})",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": dtype, "data": DATA.format(cfg),
            "config": {"workload": args.workload, "n": n, "precision": prec, "terms_per_step": terms_total,
                       "l2": "flushed between steps (256 MiB write)",
                       "prefix_classes_per_rank": f"{chi - clo} of 2^{k}" if world > 1 else "all",
                       "parallelism": f"prefix-class shards x{world}"},
            "e2e": {"value": terms_total / (e2e_step * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": h2d_step, "d2h_bytes_per_step": d2h_step, "ms_per_step": e2e_step},
            "gpu_launches": int(launches) * args.steps,
            "kernel_ms_per_step": kstep_ms,
            "result": {"value": result["value"], "words": list(result["words"]),
                       "sum_abs_terms": result["sum_abs_terms"], "cancellation_bits": result["cancellation_bits"]},
            "clocks": clk.summary(),
            "wall_s_timed": wall_steps,
        }
        if roof:
            line["roofline"] = roof
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
