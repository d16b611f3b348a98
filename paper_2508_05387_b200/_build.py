"""In-tree build of libecho.so (the product) for sm_100a with nvcc.  No JIT, no torch extension cache:
the .so lives next to this file so that it travels to the GPU box with the repository snapshot."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libecho.so")
TRACE_LIB = os.path.join(PKG, "libecho_trace.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]
LIBS: list[str] = []   # no library GEMMs: every product runs on libecho's own tcgen05 kernels


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))) + \
        [os.path.join(INCLUDE, "echo.h")]


def up_to_date(lib=LIB):
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """Build libecho.so (or, with trace=True, the diagnostic libecho_trace.so with -DECHO_TRACE)."""
    lib = TRACE_LIB if trace else LIB
    if not force and up_to_date(lib):
        return lib
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, *FLAGS, *(["-DECHO_TRACE"] if trace else []), "-I", INCLUDE, "-I", CSRC, "-o", tmp,
           *sources(), *LIBS]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed ({r.returncode}):\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if not trace:
        os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)    # git-ignored: register / spill report per build
        with open(os.path.join(ROOT, "build", "ptxas_info.txt"), "w") as f:
            f.write(r.stderr)
    if verbose:
        print(r.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force=True, verbose=True))
