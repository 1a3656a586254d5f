"""Attribute ncu per-instruction samples of the dd subtree kernel to outermost engine.cu lines
(using nvdisasm -gi inline info).  usage: python tools/sass_regions.py REPORT CUBIN_DIS KERNEL_SUBSTR"""
import collections, csv, io, re, subprocess, sys

rep, dis, ksub = sys.argv[1], sys.argv[2], sys.argv[3]
lines = open(dis).read().split("\n")
# find function section
start = None
for i, l in enumerate(lines):
    if l.startswith(".text.") and ksub in l:
        start = i
        break
insts = []
cur = None
for l in lines[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        chain = [(m.group(1).split("/")[-1], int(m.group(2)))]
        for f, ln in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3)):
            chain.append((f.split("/")[-1], int(ln)))
        cur = chain
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        insts.append((cur, l.strip()))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(src)))
hdr = r[1]
ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)")
prof = [(int(x[ie]) if x[ie].isdigit() else 0, int(x[ss]) if x[ss].isdigit() else 0) for x in r[2:]]
print("sass insts (nvdisasm)", len(insts), "ncu rows", len(prof))
agg = collections.defaultdict(lambda: [0, 0])
ts = sum(p[1] for p in prof)
for (chain, txt), (n, s) in zip(insts, prof):
    key = "?"
    if chain:
        # outermost engine.cu frame
        eng = [c for c in chain if c[0] == "engine.cu"]
        key = f"engine.cu:{eng[-1][1]}" if eng else f"{chain[-1][0]}:{chain[-1][1]}"
    agg[key][0] += s
    agg[key][1] += n
for k, (s, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 30]:
    print(f"{k:22s} samples {100*s/ts:5.1f}%  inst {n:.3e}")
