"""A/B experiments: link libgs variants that differ in one source file, for GS_LIB=<path>.
usage: python tools/variant_build.py <source-name> name=path.cu [name=path.cu ...]
(e.g. bucket.cu v1=/tmp/v1.cu); the other objects come from the release build (build/)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_11700_b200 import build as B  # noqa: E402


def main():
    src, pairs = sys.argv[1], sys.argv[2:]
    B.build()
    outdir = os.path.join(B.HERE, "build", "variants")
    os.makedirs(outdir, exist_ok=True)
    objs = [os.path.join(B.BUILD, s.replace(".cu", ".o")) for s in B.SOURCES if s != src]
    for p in pairs:
        name, path = p.split("=", 1)
        obj = os.path.join(outdir, f"{name}.o")
        cmd = [B.nvcc(), *B.ARCH, *B.COMMON, *B.PER_FILE.get(src, []), "-I", B.CSRC, "-c", path, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stdout + r.stderr)
        lib = os.path.join(outdir, f"libgs_{name}.so")
        r = subprocess.run([B.nvcc(), *B.ARCH, "-shared", "-o", lib, *objs, obj, "-lcudart"], capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stdout + r.stderr)
        print(lib)


if __name__ == "__main__":
    main()
