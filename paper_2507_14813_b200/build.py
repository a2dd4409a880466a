"""Build libmayura.so in-tree: nvcc, sm_100a only (the .so travels to the GPU box).

    python paper_2507_14813_b200/build.py [--force] [--ptxas-v]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libmayura.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "mayura.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, ptxas_verbose: bool = False, variant: str = "", defines=()) -> str:
    """variant: build lib/libmayura_<variant>.so with extra -D defines (A/B builds, loaded through
    MAYURA_LIB_PATH); the default library is lib/libmayura.so."""
    lib = LIB if not variant else os.path.join(os.path.dirname(LIB), "libmayura_%s.so" % variant)
    if not variant and not force and not _stale():
        return LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    tmp = lib + ".tmp%d" % os.getpid()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3,-pthread",
           *["-D" + d for d in defines],
           "-I", os.path.join(ROOT, "include"), "-o", tmp, *sources(), "-lpthread"]
    if ptxas_verbose:
        cmd[1:1] = ["-Xptxas", "-v"]
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else ""
    defs = [a[2:] for a in sys.argv if a.startswith("-D")]
    print(build(force="--force" in sys.argv, ptxas_verbose="--ptxas-v" in sys.argv, variant=var, defines=defs))
