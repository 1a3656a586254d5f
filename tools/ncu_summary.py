"""Summarise an ncu report: key metrics + per-execution-count SASS groups."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
want = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "smsp__thread_inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second"]
for row in rows[2:]:
    d = dict(zip(h, row))
    print(d.get("Kernel Name", "")[:80])
    for k in want:
        if k in d:
            print(f"  {k:90s} {d[k]} {dict(zip(h, u)).get(k, '')}")
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(src)))
    hdr = r[1]
    ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)"); so = hdr.index("Source")
    g = collections.defaultdict(lambda: [0, 0, 0, 0])
    ts = ti = 0
    for x in r[2:]:
        try:
            n = int(x[ie]); s = int(x[ss])
        except (ValueError, IndexError):
            continue
        op = x[so].split()
        op = (op[1] if op and op[0].startswith("@") and len(op) > 1 else (op[0] if op else ""))
        gg = g[n]; gg[0] += 1; gg[1] += s; gg[2] += n
        if op.startswith("D"):
            gg[3] += n
        ts += s; ti += n
    print("total samples", ts, "warp inst", ti)
    for n, (c, s, i, di) in sorted(g.items(), key=lambda kv: -kv[1][1])[:int(sys.argv[2])]:
        print(f"  exec={n:>12} ninstr={c:5d} samples={100*s/ts:5.1f}% inst={100*i/ti:5.1f}% fp64={di/max(i,1):.2f}")
