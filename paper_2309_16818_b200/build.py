"""Builds libmem.so (the sm_100a C-ABI library) in-tree with nvcc.

Flags: -fmad=false keeps every fp32/fp64 multiply-add unfused so the kernels
follow the written operation order; IEEE division/sqrt and no FTZ are nvcc's defaults and
--use_fast_math is never used.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmem.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# NCCL 2.28 (the copy torch ships in the venv; the system 2.27 is the fallback), for the
# sharded big map's band exchange
_VENV_NCCL = os.path.join(sys.prefix, "lib", f"python{sys.version_info[0]}.{sys.version_info[1]}", "site-packages",
                          "nvidia", "nccl")
NCCL_DIR = os.environ.get("MEM_NCCL_DIR", _VENV_NCCL if os.path.isdir(_VENV_NCCL) else "/usr")
NCCL_INC = os.path.join(NCCL_DIR, "include")
NCCL_LIB = os.path.join(NCCL_DIR, "lib") if os.path.isdir(os.path.join(NCCL_DIR, "lib")) else "/usr/lib/x86_64-linux-gnu"
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--extended-lambda", "-shared",
         "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden", "-Xptxas", "-warn-spills",
         "-I", os.path.join(ROOT, "include"), "-I", NCCL_INC]
LIBS = ["-L", NCCL_LIB, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + NCCL_LIB]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "mem.h"),
                                                                       __file__]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    extra = os.environ.get("MEM_NVCC_EXTRA", "").split()  # tuning experiments only (e.g. -DMEM_POINTS_MINB=4)
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-o", LIB + ".tmp", *sources(), *LIBS]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_variant(out, defines):
    """A copy of libmem built with other launch configurations (compile-time -D macros) at
    `out` -- for the launch-configuration invariance test only; the shipped library is LIB."""
    cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-o", out, *sources(), *LIBS]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
