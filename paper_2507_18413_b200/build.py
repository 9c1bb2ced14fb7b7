"""Build the CUDA library in-tree: paper_2507_18413_b200/libct_b200.so (sm_100a).

    python -m paper_2507_18413_b200.build [--force] [--verbose]

nvcc -gencode arch=compute_100a,code=sm_100a, -lineinfo for ncu source
correlation; links NCCL from the same wheel PyTorch loads (one libnccl.so.2 per
process).  The CUDA runtime is linked statically so the library does not
depend on which libcudart the host process loaded first.
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
LIB = os.path.join(PKG, "libct_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    try:
        import nvidia.nccl as nn  # namespace package shipped with torch
        base = list(nn.__path__)[0]
    except Exception:  # pragma: no cover
        base = None
    if base and os.path.exists(os.path.join(base, "include", "nccl.h")):
        return os.path.join(base, "include"), os.path.join(base, "lib")
    for inc in ("/usr/include", "/usr/local/include"):
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, "/usr/lib/x86_64-linux-gnu"
    raise RuntimeError("nccl.h not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(INCLUDE, "ct.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None, out: str | None = None) -> str:
    """out: build a variant library there instead (experiments; always rebuilt)."""
    if out is None and not force and not needs_build():
        return LIB
    target = out or LIB
    inc, libdir = nccl_paths()
    tmp = target + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", INCLUDE, "-I", CSRC, "-I", inc,
           os.path.join(CSRC, "ct_runtime.cu"),
           "-o", tmp, "-L", libdir, "-l:libnccl.so.2", f"-Xlinker=-rpath={libdir}",
           *(extra or [])]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
