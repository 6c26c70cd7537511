"""Build libgs.so (sm_100a) in-tree with nvcc. No torch involvement (plain C ABI)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgs.so")
OUT_DEBUG = os.path.join(HERE, "libgs_debug.so")   # -DGS_DEBUG=1: output invariant checks (csrc/debug.cu)
BUILD = os.path.join(HERE, "build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]
# projection decides integers (depth key, rect, radius) and must be bit-exact with the oracle:
# no FMA contraction, IEEE division and sqrt
PER_FILE = {"project.cu": ["-fmad=false", "-prec-div=true", "-prec-sqrt=true"]}
SOURCES = ["abi.cu", "project.cu", "binsort.cu", "bucket.cu", "bincoop.cu", "render.cu", "optim.cu", "debug.cu"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def _build_one(out: str, objdir: str, extra: list[str], force: bool, verbose: bool) -> str:
    os.makedirs(objdir, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "gs.h")]
    newest = max(os.path.getmtime(d) for d in deps)
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    from concurrent.futures import ThreadPoolExecutor

    def one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        cmd = [nvcc(), *ARCH, *COMMON, *extra, *PER_FILE.get(src, []), "-c", os.path.join(CSRC, src), "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)
    objs = []
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        for src, obj, r in ex.map(one, SOURCES):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(obj)
    cmd = [nvcc(), *ARCH, "-shared", "-o", out, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    return out


def build(force: bool = False, verbose: bool = False, debug: bool = True) -> str:
    """libgs.so (release) and libgs_debug.so (GS_DEBUG=1 checks; loaded when the environment sets
    GS_DEBUG=1)."""
    out = _build_one(OUT, BUILD, [], force, verbose)
    if debug:
        _build_one(OUT_DEBUG, os.path.join(BUILD, "debug"), ["-DGS_DEBUG=1"], force, verbose)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
