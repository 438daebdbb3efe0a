"""Build libvtrans_gpu.so in-tree (paper_2109_10433_b200/lib/) with nvcc.

    python -m paper_2109_10433_b200.build [--force] [--verbose]

Every CUDA translation unit is compiled for sm_100a only
(-gencode arch=compute_100a,code=sm_100a) with -lineinfo, so ncu's source view
maps to the kernels.  The CUDA runtime is linked statically, so the library
does not depend on which libcudart a host process (e.g. torch) carries.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(LIBDIR, "libvtrans_gpu.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["k_utf8.cu", "k_utf16.cu", "k_batch.cu", "k_datagen.cu", "k_stream.cu", "runtime.cu"]
CXX_SOURCES = ["shim.cpp"]
HEADERS = ["vt_device.cuh", "vt_kernels.h", "vt_gen.cuh", "vt_pipeline.cuh", "vt_swar.cuh"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libvtrans_gpu")


def _deps() -> list[str]:
    inc = os.path.join(ROOT, "include")
    files = [os.path.join(CSRC, f) for f in CU_SOURCES + CXX_SOURCES + HEADERS]
    for dp, _, fs in os.walk(inc):
        files += [os.path.join(dp, f) for f in fs]
    files.append(os.path.abspath(__file__))
    return files


STAMP = os.path.join(LIBDIR, "build_flags.txt")


def _flags() -> str:
    """The flags that change the build (an experimental VT_NVCC_EXTRA build
    must never pass for the product library)."""
    return " ".join([*ARCH, os.environ.get("VT_NVCC_EXTRA", "")]).strip()


def up_to_date() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return False
    with open(STAMP) as f:
        if f.read() != _flags():
            return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(f) <= t for f in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    nv = nvcc()
    common = ["-O3", "-std=c++20", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
    common += os.environ.get("VT_NVCC_EXTRA", "").split()
    cmds = []
    objs = []
    for src in CU_SOURCES:
        obj = os.path.join(OBJDIR, src + ".o")
        objs.append(obj)
        cmds.append([nv, *ARCH, *common, "-lineinfo", "-Xptxas", "-v", "--expt-relaxed-constexpr",
                     "-c", os.path.join(CSRC, src), "-o", obj])
    for src in CXX_SOURCES:
        obj = os.path.join(OBJDIR, src + ".o")
        objs.append(obj)
        cmds.append([nv, *common, "-x", "c++", "-c", os.path.join(CSRC, src), "-o", obj])

    def run(cmd):
        p = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, p

    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        for cmd, p in ex.map(run, cmds):
            logs.append(p.stdout + p.stderr)
            if p.returncode != 0:
                sys.stderr.write(" ".join(cmd) + "\n" + p.stdout + p.stderr)
                raise RuntimeError(f"nvcc failed on {cmd[-3]}")
    with open(os.path.join(LIBDIR, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    link = [nv, *ARCH, "-shared", "-cudart", "static", "-o", LIB + ".tmp", *objs,
            "-Xlinker", "-Bsymbolic", "-lpthread"]
    p = subprocess.run(link, capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(" ".join(link) + "\n" + p.stdout + p.stderr)
        raise RuntimeError("link of libvtrans_gpu.so failed")
    os.replace(LIB + ".tmp", LIB)
    with open(STAMP, "w") as f:
        f.write(_flags())
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
