"""Commit the SASS of the DD/QD inner loops (north_star item 3): profiles/sass/.

    python tools/sass_commit.py            # after python -m paper_2009_01177_b200._build

Writes
  profiles/sass/prims_<probe>.sass   cuobjdump -sass of the arithmetic probes of
                                     tools/probes/prims.cu (rank2 / vec / pivot / leaf /
                                     accumulate for fp64, DD and QD; same flags as the engine)
  profiles/sass/subtree_kernel_dd.sass   the headline kernel as shipped in libtor_b200.so
  profiles/sass/counts.json          FP64 instruction counts (DFMA, DADD, DMUL, MUFU) and
                                     instruction totals of every probe and of every engine
                                     kernel, with the sha256 of the sources they came from
tests/test_sass.py recomputes all of it from the sources / the built library and compares.
"""
from __future__ import annotations

import hashlib
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "sass")
LIB = os.path.join(ROOT, "paper_2009_01177_b200", "libtor_b200.so")
PROBES = os.path.join(ROOT, "tools", "probes", "prims.cu")
SOURCES = ["paper_2009_01177_b200/csrc/arith.cuh", "paper_2009_01177_b200/csrc/engine.cu",
           "paper_2009_01177_b200/csrc/engine.cuh", "tools/probes/prims.cu"]
OPS = ("DFMA", "DADD", "DMUL", "MUFU")
INSN = re.compile(r"^\s+/\*[0-9a-f]{4,5}\*/\s+(?:@!?U?P[T\d]\s+)?([A-Z0-9_]+)")


def sources_sha() -> str:
    h = hashlib.sha256()
    for s in SOURCES:
        h.update(open(os.path.join(ROOT, s), "rb").read())
    return h.hexdigest()


def split_functions(sass: str) -> dict[str, list[str]]:
    out, cur = {}, None
    for line in sass.split("\n"):
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            out[cur] = []
            continue
        if cur is not None:
            out[cur].append(line)
    return out


def count(lines) -> dict:
    c = {k: 0 for k in OPS}
    total = 0
    for ln in lines:
        m = INSN.match(ln)
        if not m:
            continue
        total += 1
        op = m.group(1).split(".")[0]
        if op in c:
            c[op] += 1
    c["total"] = total
    return c


def probe_sass() -> str:
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "p.cubin")
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false", "-std=c++17",
                        "-DTOR_QD_RANK_INLINE", "-cubin", "-o", out, PROBES], check=True)
        return subprocess.run(["cuobjdump", "-sass", out], capture_output=True, text=True, check=True).stdout


def engine_sass() -> str:
    return subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout


KERNELS = ("fold_pass_kernel", "small_job_kernel", "subtree_kernel", "direct_prefix_kernel", "make_jobs_kernel",
           "prefix_level_kernel", "fixed_fold_kernel", "fixed_kernel")


def short(name: str) -> str:
    """Readable kernel name: subtree_kernel<dd>, small_job_kernel<qd,7>, fixed_kernel<2> ..."""
    for kn in KERNELS:
        tag = f"{len(kn)}{kn}I"
        if tag in name:
            rest = name.split(tag, 1)[1]
            kind = ("dd" if rest.startswith("NS_2dd") else "qd" if rest.startswith("NS_2qd")
                    else "fp64" if rest.startswith("d") else "")
            lit = re.match(r"(?:NS_2[dq]dE|d)?Li(\d+)E", rest) or re.match(r"Li(\d+)E", rest)
            args = ",".join(x for x in (kind, lit.group(1) if lit else "") if x)
            return f"{kn}<{args}>"
    return name


def collect():
    probes = {k: count(v) for k, v in split_functions(probe_sass()).items()}
    eng = {short(k): count(v) for k, v in split_functions(engine_sass()).items()}
    return probes, eng


def main():
    os.makedirs(OUT, exist_ok=True)
    ps = split_functions(probe_sass())
    for name, lines in ps.items():
        with open(os.path.join(OUT, f"prims_{name}.sass"), "w") as f:
            f.write(f"// cuobjdump -sass of probe {name} (tools/probes/prims.cu, sm_100a)\n" + "\n".join(lines) + "\n")
    es = split_functions(engine_sass())
    for name, lines in es.items():
        if short(name) == "subtree_kernel<dd>":
            with open(os.path.join(OUT, "subtree_kernel_dd.sass"), "w") as f:
                f.write(f"// cuobjdump -sass of {name} in libtor_b200.so (sm_100a)\n" + "\n".join(lines) + "\n")
    rec = {"note": __doc__.strip().split("\n")[0], "sources_sha256": sources_sha(), "sources": SOURCES,
           "probes": {k: count(v) for k, v in ps.items()},
           "engine": {short(k): count(v) for k, v in es.items()}}
    json.dump(rec, open(os.path.join(OUT, "counts.json"), "w"), indent=1, sort_keys=True)
    print(json.dumps(rec["engine"], indent=1)[:3000])


if __name__ == "__main__":
    sys.exit(main())
