"""In-tree build of libtor_b200.so (sm_100a) -- no JIT cache, the .so travels with the repo.

    python -m paper_2009_01177_b200._build
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
BUILD = os.environ.get("TOR_BUILD_DIR") or os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libtor_b200.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                     "-Xptxas", "-v", "-diag-suppress", "177"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall"]


def cuda_home() -> str:
    for c in (os.environ.get("CUDA_HOME"), "/usr/local/cuda"):
        if c and os.path.exists(os.path.join(c, "bin", "nvcc")):
            return c
    nv = shutil.which("nvcc")
    if nv:
        return os.path.dirname(os.path.dirname(nv))
    raise RuntimeError("nvcc not found")


def _run(cmd, log):
    p = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
    if p.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    return p


def _sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    srcs = _sources() + [os.path.join(os.path.dirname(PKG), "include", "tor_capi.h"), __file__]
    return all(os.path.getmtime(s) <= t for s in srcs)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    lib_path = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    ch = cuda_home()
    nvcc = os.path.join(ch, "bin", "nvcc")
    inc = ["-I" + os.path.join(ch, "include"), "-I" + os.path.join(os.path.dirname(PKG), "include")]
    os.makedirs(BUILD, exist_ok=True)
    jobs = [
        ([nvcc] + NVCC_FLAGS + [f"-D{d}" for d in defines] + inc + ["-c", os.path.join(CSRC, "engine.cu"), "-o", os.path.join(BUILD, "engine.o")],
         os.path.join(BUILD, "engine.log")),
        ([nvcc] + NVCC_FLAGS + inc + ["-c", os.path.join(CSRC, "fixed.cu"), "-o", os.path.join(BUILD, "fixed.o")],
         os.path.join(BUILD, "fixed.log")),
        (["g++"] + CXX_FLAGS + inc + ["-c", os.path.join(CSRC, "host.cpp"), "-o", os.path.join(BUILD, "host.o")],
         os.path.join(BUILD, "host.log")),
        (["g++"] + CXX_FLAGS + [f"-D{d}" for d in defines] + inc + ["-c", os.path.join(CSRC, "capi.cpp"), "-o", os.path.join(BUILD, "capi.o")],
         os.path.join(BUILD, "capi.log")),
        (["g++"] + CXX_FLAGS + inc + ["-c", os.path.join(CSRC, "gbsa.cpp"), "-o", os.path.join(BUILD, "gbsa.o")],
         os.path.join(BUILD, "gbsa.log")),
    ]
    with ThreadPoolExecutor(len(jobs)) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    tmp = lib_path + ".tmp"
    _run([nvcc] + ARCH + ["-shared", "-o", tmp, os.path.join(BUILD, "engine.o"), os.path.join(BUILD, "fixed.o"),
                          os.path.join(BUILD, "host.o"), os.path.join(BUILD, "gbsa.o"),
                          os.path.join(BUILD, "capi.o"), "-lcudart_static", "-lrt", "-lpthread", "-ldl"],
         os.path.join(BUILD, "link.log"))
    os.replace(tmp, lib_path)
    if verbose:
        print(open(os.path.join(BUILD, "engine.log")).read())
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
