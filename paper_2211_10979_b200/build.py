"""Build libsimplex.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension).

    python -m paper_2211_10979_b200.build [--force]

The shared library links the CUDA runtime statically and NCCL dynamically (the
torch-bundled NCCL 2.28 under site-packages/nvidia/nccl, found at build time and
recorded as an rpath)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsimplex.so")
SOURCES = [os.path.join(CSRC, f) for f in ("kernels.cu", "engine.cpp", "host_lane.cpp")]
DEPS = SOURCES + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
    [os.path.join(ROOT, "include", "libsimplex.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    """(include_dir, lib_dir) of the NCCL that torch uses."""
    cands = []
    try:
        import nvidia.nccl as nn  # type: ignore
        cands += [os.path.dirname(p) if p.endswith("__init__.py") else p for p in list(nn.__path__)]
    except Exception:
        pass
    for sp in sys.path:
        cands.append(os.path.join(sp, "nvidia", "nccl"))
    for d in cands:
        inc, lib = os.path.join(d, "include"), os.path.join(d, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
            return inc, lib
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr/include", "/usr/lib/x86_64-linux-gnu"
    raise RuntimeError("nccl.h not found")


def nvcc():
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if p and os.path.exists(p):
            return p
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compile libsimplex.so (or, for experiments, a variant with extra -D `defines` at `out`)."""
    if not force and not defines and out is None and up_to_date():
        return LIB
    target = out or LIB
    inc, lib = nccl_dirs()
    ncclso = sorted(glob.glob(os.path.join(lib, "libnccl.so*")))[0]
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xptxas", "-v",
           "-Xcompiler", "-fPIC,-O2,-ffp-contract=off,-fopenmp", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
           *["-D" + d for d in defines], *SOURCES, "-o", target + ".tmp",
           "-L", lib, "-l:" + os.path.basename(ncclso), "-Xlinker", "-rpath," + lib, "-lgomp"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + res.stdout + res.stderr)
    if verbose:
        print(res.stderr)
    if out is None:
        with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
            f.write(res.stderr)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
