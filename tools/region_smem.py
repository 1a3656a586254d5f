"""Shared-memory wavefronts (actual / ideal) per engine.cu region of an ncu report.
usage: python tools/region_smem.py REPORT DISASM_TXT [kernel_substr]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, dis = sys.argv[1], sys.argv[2]
ksub = sys.argv[3] if len(sys.argv) > 3 else "subtree_kernelINS_2dd"
lines = open(dis).read().split("\n")
st = [i for i, l in enumerate(lines) if l.startswith(".text.") and ksub in l][0]
insts, cur, fresh = [], [], True
for l in lines[st + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if fresh:
            cur, fresh = [], False
        cur.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    mm = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s*(.*)", l)
    if mm:
        insts.append((list(cur), mm.group(2)))
        fresh = True
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
h = r[1]
rows = r[2:]
iw, ii = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Ideal")
agg = collections.defaultdict(lambda: [0, 0])
for (chain, txt), row in zip(insts, rows):
    eng = [c for c in chain if c[0] == "engine.cu"]
    k = eng[-1][1] if eng else 0
    agg[k][0] += int(row[iw] or 0)
    agg[k][1] += int(row[ii] or 0)
tot = sum(v[0] for v in agg.values())
for k, (a, b) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:10]:
    print(f"line {k:5d} wavefronts {a/1e9:6.2f}e9 ({100*a/tot:4.1f}%)  ideal {b/1e9:6.2f}e9  x{a/max(b,1):.2f}")
