"""Per-region executed-instruction mix (thread instructions / terms) of an ncu report.

usage: python tools/region_ops.py REPORT DISASM_TXT N_MODES [kernel_substr]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, dis, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
ksub = sys.argv[4] if len(sys.argv) > 4 else "subtree_kernelINS_2dd"
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text.") and ksub in l][0]
insts, cur, fresh = [], [], True
for l in lines[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if fresh:
            cur, fresh = [], False
        cur.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    mm = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s*(.*)", l)
    if mm:
        op = mm.group(1).split()
        op = op[1] if op and op[0].startswith("@") else (op[0] if op else "")
        insts.append((list(cur), op.split(".")[0]))
        fresh = True
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
hdr = r[1]
ie = hdr.index("Predicated-On Thread Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
rows = r[2:]
assert len(rows) == len(insts)
agg = collections.defaultdict(collections.Counter)
samp = collections.Counter()
for (chain, op), row in zip(insts, rows):
    eng = [c for c in chain if c[0] == "engine.cu"]
    key = eng[-1][1] if eng else 0
    agg[key][op] += int(row[ie] or 0)
    samp[key] += int(row[ss] or 0)
T = float(2 ** n)
tot = sum(samp.values())
for key in sorted(agg, key=lambda k: -samp[k])[:9]:
    c = agg[key]
    allv = sum(c.values()) / T
    fp = sum(v for o, v in c.items() if o in ("DFMA", "DADD", "DMUL")) / T
    print(f"line {key:5d} {100*samp[key]/tot:5.1f}%  inst/term {allv:6.1f}  fp64 {fp:6.1f}  | " +
          " ".join(f"{o}:{v/T:.1f}" for o, v in c.most_common(9)))
