"""Build libgpart.so (sm_100a) in-tree with nvcc.

``python -m paper_2105_10312_b200._build`` or ``__graft_entry__.build()``.
The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUT = os.path.join(PKG, "libgpart.so")
BUILD = os.path.join(PKG, "build")

SOURCES = ["abi.cu", "generate.cu", "enumerate.cu", "wcet.cu", "exhaustive.cu", "allocate.cu",
           "ratio.cu", "threshold.cu", "allocate_big.cu", "exhaustive_bp.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-I", INCLUDE, "-I", CSRC]


def _deps_mtime():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "gpart.h"),
                                                                  __file__]
    return max(os.path.getmtime(f) for f in files)


def _compile(src, verbose, bdir=BUILD, extra=()):
    obj = os.path.join(bdir, src.replace(".cu", ".o"))
    cmd = ["nvcc", *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, out: str = OUT, extra=()) -> str:
    """Build libgpart.so; `out` / `extra` (nvcc -D flags) make A/B variants of the library
    (loaded through GP_LIB) without touching the default build."""
    if not force and os.path.exists(out) and os.path.getmtime(out) >= _deps_mtime():
        return out
    bdir = BUILD if out == OUT else out + ".build"
    os.makedirs(bdir, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose, bdir, extra), SOURCES))
    if verbose:
        for obj, log in results:
            sys.stderr.write(f"== {os.path.basename(obj)}\n{log}")
    tmp = out + ".tmp"
    subprocess.check_call(["nvcc", *ARCH, "-shared", "-o", tmp, *[o for o, _ in results]])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    # python -m paper_2105_10312_b200._build [--force] [-v] [--out PATH -DNAME=VAL ...]
    args = sys.argv[1:]
    out = args[args.index("--out") + 1] if "--out" in args else OUT
    print(build(force="--force" in args, verbose="-v" in args, out=out,
                extra=[a for a in args if a.startswith("-D")]))
