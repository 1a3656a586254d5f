"""Write profiles/sass_counts.json from an ncu --set full report of the subtree kernel.

usage: python tools/sass_counts.py REPORT.ncu-rep N_MODES MODE [SOURCE_CMD]
Per-term counts = executed predicated-on thread instructions / 2^n (terms in one
launch of the n-mode engine); flops = 2*DFMA + DADD + DMUL.  bench.py reads the
file for its roofline (FP64-pipe bound)."""
import csv
import io
import json
import os
import subprocess
import sys

rep, n, mode = sys.argv[1], int(sys.argv[2]), sys.argv[3]
cmd = sys.argv[4] if len(sys.argv) > 4 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
best = None
for row in rows[2:]:
    d = dict(zip(h, row))
    if "subtree_kernel" not in d.get("Kernel Name", ""):
        continue
    t = float(d["gpu__time_duration.sum"].replace(",", ""))
    if best is None or t > best[0]:
        best = (t, d)
if best is None:
    sys.exit("no subtree_kernel launch in report")
t, d = best
units = dict(zip(h, rows[1]))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
f = lambda k: float(d[k].replace(",", "")) * SCALE.get(units.get(k, ""), 1)
terms = float(2 ** n)
dfma = f("sm__sass_thread_inst_executed_op_dfma_pred_on.sum") / terms
dadd = f("sm__sass_thread_inst_executed_op_dadd_pred_on.sum") / terms
dmul = f("sm__sass_thread_inst_executed_op_dmul_pred_on.sum") / terms
unit = [x for x in rows[1]][h.index("gpu__time_duration.sum")]
ms = t / 1e6 if unit == "ns" else (t / 1e3 if unit in ("us", "usecond") else t)
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "sass_counts.json")
out = json.load(open(path)) if os.path.exists(path) else {}
out.update({
    "note": "FP64 work per subset-term of the engine's subtree kernel from an ncu --set full capture: "
            "executed predicated-on thread instructions / 2^n terms; flops = 2*DFMA + DADD + DMUL. "
            "Written by tools/sass_counts.py.",
    "round": 1,
})
out.setdefault(mode, {})
out[mode] = {"dfma": dfma, "dadd": dadd, "dmul": dmul, "fp64_instr": dfma + dadd + dmul,
             "n": n, "source": os.path.basename(rep), "cmd": cmd,
             "kernel_ms": ms,
             "dram_bytes_per_launch": f("dram__bytes_read.sum") + f("dram__bytes_write.sum"),
             "fp64_pipe_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")}
out.setdefault("flops_per_term", {})[mode] = 2 * dfma + dadd + dmul
out.setdefault("dram_bytes_per_launch", {})[mode] = out[mode]["dram_bytes_per_launch"]
out.setdefault("kernel_ms", {})
if not isinstance(out["kernel_ms"], dict):
    out["kernel_ms"] = {}
out["kernel_ms"][mode] = ms
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
