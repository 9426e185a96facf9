"""Build libarrabit.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python paper_1507_06078_b200/build.py [--verbose]     (or __graft_entry__.build())
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["spmm_kernels.cu", "stencil_kernels.cu", "dense_kernels.cu", "comm.cu", "api.cu"]
LIB = os.path.join(HERE, "libarrabit.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> str:
    """NCCL shipped with torch (the one torch.distributed loads): headers + libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    return "/usr"


NCCL = _nccl_dir()
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, "internal.cuh"), __file__,
                                                         os.path.join(HERE, "..", "include", "arrabit.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile the CUDA sources into ``out`` (default: the in-tree libarrabit.so).
    ``defines``: extra -D macros (used for tuning variants)."""
    lib = out or LIB
    if out is None and not force and not _stale():
        return LIB
    objs = []
    for s in SOURCES:
        obj = os.path.join(CSRC, s.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, f"-I{NCCL}/include", *[f"-D{d}" for d in defines], "-c", os.path.join(CSRC, s), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *objs,
           "-lcusolver", "-lcudart", f"-L{NCCL}/lib", "-l:libnccl.so.2", f"-Xlinker=-rpath,{NCCL}/lib"]
    subprocess.check_call(cmd)
    for o in objs:
        os.remove(o)
    return lib


CHECKED = os.path.join(HERE, "libarrabit_checked.so")


def build_checked() -> str:
    """The bounds-checked variant (-DARR_CHECK_BOUNDS: device checks that trap)."""
    return build(out=CHECKED, defines=["ARR_CHECK_BOUNDS"])


if __name__ == "__main__":
    if "--checked" in sys.argv:
        print(build_checked())
    else:
        build(force=True, verbose="--verbose" in sys.argv)
        print(LIB)
