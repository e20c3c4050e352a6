"""Build libmist.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2503_19050_b200.build

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; no fast-math
(IEEE fp64 division and rounding are part of the parity contract).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libmist.so")
BUILD = os.path.join(PKG, "_build")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch's bundled NCCL (same soname torch loads)
        base = list(nn.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = _sources() + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(INCLUDE, "mist.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "", defs=None) -> str:
    """variant "counters": instrumented copy libmist_counters.so (-DMIST_COUNTERS,
    event counters printed by the sweep); any other variant name with `defs`
    (-D flags): an A/B copy ab/libmist_<variant>.so.  The product library is
    untouched by variants."""
    lib_path, build_dir = LIB, BUILD
    defs = list(defs or [])
    if variant == "counters":
        lib_path, build_dir, defs = os.path.join(PKG, "libmist_counters.so"), BUILD + "_counters", ["-DMIST_COUNTERS"]
        force = True
    elif variant:
        os.makedirs(os.path.join(ROOT, "ab"), exist_ok=True)
        lib_path, build_dir = os.path.join(ROOT, "ab", f"libmist_{variant}.so"), BUILD + "_" + variant
        force = True
    if not force and not _stale():
        return LIB
    os.makedirs(build_dir, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    objs = []
    for src in _sources():
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        if src.endswith(".cu"):
            cmd = ["nvcc", *ARCH, *defs, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v" if verbose else "-O3", "-I", INCLUDE, "-I", CSRC, "-I", nccl_inc,
                   "-c", src, "-o", obj]
        else:
            cmd = ["g++", *defs, "-O2", "-std=c++17", "-fPIC", "-fopenmp", "-I", INCLUDE, "-I", CSRC,
                   "-I", "/usr/local/cuda/include", "-I", nccl_inc, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib_path + ".tmp"
    cmd = ["nvcc", *ARCH, "-shared", "-o", tmp, *objs, "-L", nccl_lib, "-l:libnccl.so.2", "-lgomp",
           "-Xlinker", "-rpath," + nccl_lib, "-cudart", "static"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    variant = "counters" if "--counters" in sys.argv else ""
    if "--variant" in sys.argv:
        variant = sys.argv[sys.argv.index("--variant") + 1]
    build(force="--force" in sys.argv, verbose="--quiet" not in sys.argv, variant=variant,
          defs=[a for a in sys.argv[1:] if a.startswith("-D")])
