"""Compile libtpq.so (sm_100a CUDA kernels + C++ host half of the C-ABI) in-tree with nvcc.

    python -m paper_2402_04925_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libtpq.so")
SOURCES = ["tpq_host.cpp", "tpq_kernels.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_root() -> str:
    import nvidia.nccl  # namespace package shipped with torch's CUDA wheels (NCCL 2.28.9)
    return list(nvidia.nccl.__path__)[0]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "tpq.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, prof: bool = False, defines=(), name=None) -> str:
    """prof=True builds libtpq_prof.so with -DTPQ_PROF (per-CTA timeline, profiling only);
    `defines` + `name` build experiment variants (e.g. ablations) next to the product library."""
    lib = os.path.join(PKG, name) if name else (LIB.replace("libtpq.so", "libtpq_prof.so") if prof else LIB)
    if not force and not prof and not name and not _stale():
        return LIB
    nr = nccl_root()
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC,-O3",
           "-Xptxas", "-v" if verbose else "-O3",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nr, "include"),
           *[os.path.join(CSRC, s) for s in SOURCES],
           "-L", os.path.join(nr, "lib"), "-l:libnccl.so.2",
           f"-Xlinker=-rpath,{os.path.join(nr, 'lib')}",
           *(["-DTPQ_PROF"] if prof else []), *[f"-D{d}" for d in defines],
           "-o", lib + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if verbose:
        sys.stderr.write(r.stdout + r.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, prof="--prof" in sys.argv))
