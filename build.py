"""Build libeik.so in-tree for sm_100a (no JIT cache, no torch extension).

    python build.py [--force]
"""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1805_02144_b200")
SRC = [os.path.join(PKG, "csrc", "eik_api.cu")]
DEPS = SRC + [os.path.join(PKG, "csrc", f) for f in ("eik_dev.cuh", "eik_control.h")] + [
    os.path.join(ROOT, "include", "eik.h")]
OUT = os.path.join(PKG, "libeik.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force=False, verbose=False, out=OUT, defines=()):
    if not force and out == OUT and up_to_date():
        return OUT
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out + ".tmp", *SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(ROOT, "build", "ptxas.log" if out == OUT else os.path.basename(out) + ".ptxas.log")
    os.makedirs(os.path.dirname(log), exist_ok=True)
    with open(log, "w") as fh:
        fh.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libeik.so")
    os.replace(out + ".tmp", out)
    if verbose:
        print(r.stderr)
    return out


if __name__ == "__main__":
    if "--variant" in sys.argv:
        # python build.py --variant NAME DEF1 DEF2 ...  -> build/libeik_NAME.so
        k = sys.argv.index("--variant")
        name, defs = sys.argv[k + 1], sys.argv[k + 2:]
        print(build(force=True, out=os.path.join(ROOT, "build", f"libeik_{name}.so"),
                    defines=defs))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
