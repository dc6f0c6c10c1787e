"""In-tree build of the CUDA C-ABI library (and the test-only oracle).

``python -m paper_2007_03298_b200.build`` compiles
``paper_2007_03298_b200/libdssync_b200.so`` for sm_100a with nvcc.  The
built ``.so`` is git-ignored but travels to the GPU box with the gpurun
snapshot, so the GPU side never needs a compiler.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libdssync_b200.so")
BUILD = os.path.join(ROOT, "build", "dssync_b200")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # no FMA contraction anywhere on the parity path; the kernels
    # also use explicit __f*_rn / __d*_rn intrinsics
    "-fmad=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-O2,-Wall,-ffp-contract=off",
    "-I" + INCLUDE, "-I" + CSRC,
]

SOURCES = ["dssync_b200.cu", "engine.cu", "problems_abi.cu", "schedule.cpp", "problems.cpp"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the DS-Sync CUDA library")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_lib(force: bool = False, verbose: bool = False, ptxas_v: bool = False,
              defines: tuple = (), out: str = LIB) -> str:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "dssync_b200.h")]
    if not force and not _stale(out, deps):
        return out
    bdir = BUILD if out == LIB else os.path.join(BUILD, os.path.basename(out) + ".d")
    os.makedirs(bdir, exist_ok=True)
    nvcc = _nvcc()
    objs, cmds = [], []
    for src in SOURCES:
        obj = os.path.join(bdir, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *["-D" + d for d in defines], "-c", os.path.join(CSRC, src), "-o", obj]
        if ptxas_v and src.endswith(".cu"):
            cmd.insert(1, "-Xptxas=-v")
        if verbose:
            print(" ".join(cmd), flush=True)
        cmds.append(cmd)
        objs.append(obj)
    # the translation units are independent: compile them side by side
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c, check=True), cmds)):
            pass
    tmp = out + ".tmp"
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


def build_variant(name: str, defines: tuple) -> str:
    """Tuning builds: build/variants/libdssync_b200_<name>.so (A/B runs via DSS_LIB_VARIANT)."""
    vdir = os.path.join(ROOT, "build", "variants")
    os.makedirs(vdir, exist_ok=True)
    return build_lib(force=True, defines=defines, out=os.path.join(vdir, f"libdssync_b200_{name}.so"))


if __name__ == "__main__":
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        name, defs = sys.argv[i + 1], tuple(sys.argv[i + 2:])
        print(build_variant(name, defs))
    else:
        build_lib(force="--force" in sys.argv, verbose=True, ptxas_v="--ptxas-v" in sys.argv)
        print(LIB)
