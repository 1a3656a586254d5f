"""SASS instruction count per engine.cu call-site region of the dd subtree kernel.
usage: python tools/region_sizes.py OBJ.o [kernel_substr]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

obj = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else "subtree_kernelINS_2dd"
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
lines = txt.split("\n")
st = [i for i, l in enumerate(lines) if l.startswith(".text.") and ksub in l][0]
cur, fresh, cnt, total = [], True, collections.Counter(), 0
for l in lines[st + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        if fresh:
            cur, fresh = [], False
        cur.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
        eng = [c for c in cur if c[0] == "engine.cu"]
        cnt[eng[-1][1] if eng else 0] += 1
        total += 1
        fresh = True
print(total, "instrs;", " ".join(f"{k}:{v}" for k, v in sorted(cnt.items(), key=lambda kv: -kv[1])[:10]))
