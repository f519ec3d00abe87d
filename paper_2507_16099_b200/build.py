"""Build libfp8train.so in-tree with nvcc for sm_100a (no torch JIT, no caches).

    python paper_2507_16099_b200/build.py [-v] [-f]     # or __graft_entry__.build()

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, IEEE fp32 semantics
(-ftz=false -prec-div=true -prec-sqrt=true, never --use_fast_math: the casts must be
bit-exact, DESIGN.md R-c4/R-c6/R-c11).  Links the NCCL that the torch wheel loads
(nvidia-nccl-cu12) so there is one libnccl.so.2 in the process.
"""

import glob
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libfp8train.so")
BUILD = os.path.join(PKG, "_build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
           "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "--expt-relaxed-constexpr"]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    raise RuntimeError("nvcc not found")


def nccl_paths():
    site = sysconfig.get_paths()["purelib"]
    inc = os.path.join(site, "nvidia", "nccl", "include")
    lib = os.path.join(site, "nvidia", "nccl", "lib")
    if not os.path.exists(os.path.join(inc, "nccl.h")):
        raise RuntimeError("NCCL headers (nvidia-nccl-cu12) not found under " + site)
    return inc, lib


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale(out, deps):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False):
    nvcc = _nvcc()
    inc, lib = nccl_paths()
    os.makedirs(BUILD, exist_ok=True)
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    objs = []
    for src in sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if not force and not _stale(obj, [src] + headers):
            continue
        extra = os.environ.get("FP8T_NVCC_EXTRA", "").split()   # experiments, e.g. -DFP8T_EPI_WARPS_ACC2=4
        cmd = [nvcc] + ARCH + NVFLAGS + extra + ["-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc,
                                         "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        cmd = [nvcc] + ARCH + ["-shared", "-o", LIB] + objs + \
            ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(LIB)
