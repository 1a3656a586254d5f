"""Per-engine.cu-call-site stall breakdown of an ncu report (needs nvdisasm -gi dump).

usage: python tools/region_stalls.py REPORT DISASM_TXT [kernel_substr]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, dis = sys.argv[1], sys.argv[2]
ksub = sys.argv[3] if len(sys.argv) > 3 else "subtree_kernelINS_2dd"
lines = open(dis).read().split("\n")
start = [i for i, l in enumerate(lines) if l.startswith(".text.") and ksub in l][0]
# nvdisasm -gi prints the inline stack as successive //## lines, innermost first
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
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        insts.append(list(cur))
        fresh = True
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(src)))
hdr = r[1]
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = hdr.index("Warp Stall Sampling (All Samples)")
rows = r[2:]
assert len(rows) == len(insts), (len(rows), len(insts))
# region = outermost engine.cu line in the subtree kernel body
site = collections.defaultdict(lambda: collections.Counter())
for chain, row in zip(insts, rows):
    eng = [c for c in (chain or []) if c[0] == "engine.cu"]
    key = eng[-1][1] if eng else 0
    c = site[key]
    c["_all"] += int(row[tot] or 0)
    for i in cols:
        c[hdr[i]] += int(row[i] or 0)
grand = sum(c["_all"] for c in site.values())
for key, c in sorted(site.items(), key=lambda kv: -kv[1]["_all"])[:12]:
    top = sorted(((v, k) for k, v in c.items() if k != "_all"), reverse=True)[:6]
    print(f"line {key:5d} {100*c['_all']/grand:5.1f}%  " +
          " ".join(f"{k[6:]}:{100*v/max(1,c['_all']):.0f}" for v, k in top))

if len(sys.argv) > 4:
    # per-(inner engine.cu line) breakdown of one region
    want = int(sys.argv[4])
    sub = collections.defaultdict(collections.Counter)
    for chain, row in zip(insts, rows):
        eng = [c for c in (chain or []) if c[0] == "engine.cu"]
        if not eng or eng[-1][1] != want:
            continue
        k = eng[0][1] if len(eng) > 0 else 0
        c = sub[k]
        c["_all"] += int(row[tot] or 0)
        for i in cols:
            c[hdr[i]] += int(row[i] or 0)
    print(f"--- region {want} by innermost engine.cu line")
    for key, c in sorted(sub.items(), key=lambda kv: -kv[1]["_all"])[:25]:
        top = sorted(((v, k) for k, v in c.items() if k != "_all"), reverse=True)[:4]
        print(f"  line {key:5d} {100*c['_all']/grand:5.2f}%  " +
              " ".join(f"{k[6:]}:{100*v/max(1,c['_all']):.0f}" for v, k in top))
