"""In-tree build of the CUDA extension ``libdot_b200.so`` (sm_100a).

    python -m paper_2307_15333_b200.build [--force] [-v]

Plain nvcc, no torch extension machinery: the library exposes only the C ABI
declared in ``include/dot_b200.h`` and is loaded with ctypes.  Each source is
compiled to an object in parallel, then linked.
"""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdot_b200.so")
SOURCES = ["capi.cu", "render.cu", "sorted.cu", "refine.cu", "optim.cu", "plan.cu"]
HEADERS = ["dot_tree.cuh", "dot_exp.cuh", "dot_internal.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "dot_b200.h"))
    return any(os.path.exists(p) and os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    """Compile every source for sm_100a and link ``out``; ``defines`` adds
    -D flags (experiment variants only -- the product library uses none)."""
    if not force and not _stale(out):
        return out
    objdir = out + ".objs"
    os.makedirs(objdir, exist_ok=True)
    extra = [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-c", "-o", obj, os.path.join(CSRC, src)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        return obj, " ".join(cmd) + "\n" + res.stdout + res.stderr, res.returncode

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    log = "".join(r[1] for r in results)
    ok = all(r[2] == 0 for r in results)
    tmp = out + ".tmp"
    if ok:
        cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp,
               *[r[0] for r in results], "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log += " ".join(cmd) + "\n" + res.stdout + res.stderr
        ok = res.returncode == 0
    if out == LIB:
        with open(os.path.join(PKG, "build.log"), "w") as fh:
            fh.write(log)
    if not ok:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed building {os.path.basename(out)} (see build.log)")
    if verbose:
        sys.stdout.write(log)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
