"""Build the sm_100a shared library libsc_b200.so in-tree with nvcc (no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libsc_b200.so")
SOURCES = ["plan.cpp", "factor_plan.cpp", "kernels.cu", "factor.cu", "pcpg.cu", "api.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "sc_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str = "", defines=()) -> str:
    """out/defines: variant builds for A/B measurements (e.g. libsc_b200_wn2.so with -DSC_WN16=2)."""
    global LIB
    if out:
        LIB = os.path.join(HERE, out)
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, *[f"-D{d}" for d in defines], "-Xptxas", "-v" if verbose else "-O3",
           "-o", LIB + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES], "-lcudart", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libsc_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    # python build.py [-v] [out=libname.so] [NAME=VALUE ...]  (defines for variant builds)
    extra = [a for a in sys.argv[1:] if a != "-v"]
    outs = [a[4:] for a in extra if a.startswith("out=")]
    build(force=True, verbose="-v" in sys.argv, out=outs[0] if outs else "",
          defines=[a for a in extra if not a.startswith("out=")])
    print(LIB)
