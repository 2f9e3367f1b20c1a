"""Build libvmfa_b200.so in-tree for sm_100a (nvcc; no GPU needed).

    python -m paper_2501_12299_b200.build      # or __graft_entry__.build()

Objects go to build/, the shared library to paper_2501_12299_b200/_lib/ (git-ignored;
it travels to the GPU box with the gpurun snapshot). The CUDA runtime is linked
statically so the library does not depend on which libcudart torch loaded.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "_lib")
OBJ_DIR = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(OUT_DIR, "libvmfa_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# extra nvcc flags for diagnostic builds (e.g. -DVMFA_STATS_PROF; rebuild with force=True)
EXTRA = os.environ.get("VMFA_NVCC_EXTRA", "").split()
CU_SOURCES = ["vmfa_kernels.cu", "vmfa_score_tc.cu", "vmfa_score_ws.cu", "vmfa_fixup.cu", "vmfa_ops.cu", "vmfa_stats_tc.cu", "vmfa_sort.cu", "vmfa_capi.cu"]
CXX_SOURCES = ["host/vmfa_host.cpp", "host/vmfa_io.cpp", "host/vmfa_synth.cpp"]
DEPS_H = ["vmfa_kernels.cuh", "vmfa_internal.hpp", "vmfa_rng.hpp"]


def _newer(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    os.makedirs(OBJ_DIR, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC]
    headers = [os.path.join(CSRC, h) for h in DEPS_H] + [os.path.join(ROOT, "include", "vmfa_b200.h")]
    objs = []
    for src in CU_SOURCES + CXX_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJ_DIR, src.replace("/", "_") + ".o")
        objs.append(obj)
        if not force and not _newer(obj, [path] + headers):
            continue
        if src.endswith(".cu"):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-warn-spills", *EXTRA, *inc, "-c", path, "-o", obj]
        else:
            # -ffp-contract=off: the synthetic rows are bit-identical to the
            # oracle build of the same generator (oracle/Makefile)
            cmd = ["g++", "-O3", "-std=c++17", "-fPIC", "-pthread", "-Wall", "-Wextra", "-ffp-contract=off",
                   "-I", "/usr/local/cuda/include", *inc, "-c", path, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if force or _newer(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs, "-lpthread"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
