"""Build libgi.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libgi.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "gi.h")]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in _deps())


def build_lib(force: bool = False, verbose: bool = False) -> str:
    """gi_kernels.cu is compiled twice (CTA width 512 = primary, 1024 for skewed graphs),
    the other sources once; objects are linked into one shared library."""
    if not force and not needs_build():
        return SO
    nvcc = os.environ.get("NVCC", "nvcc")
    # -lineinfo: ncu source correlation; measured neutral on every config
    base = [nvcc, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
    if verbose:
        base.insert(1, "-Xptxas=-v")
    objdir = os.path.join(PKG, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    units = []
    for src in sources():
        name = os.path.splitext(os.path.basename(src))[0]
        if name == "gi_kernels":
            units.append((src, os.path.join(objdir, "gi_kernels_512.o"), ["-DGI_BLOCK=512", "-DGI_VARIANT=v512", "-DGI_PRIMARY=1"]))
            units.append((src, os.path.join(objdir, "gi_kernels_1024.o"),
                          ["-DGI_BLOCK=1024", "-DGI_VARIANT=v1024", "-DGI_PRIMARY=0"]))
        else:
            units.append((src, os.path.join(objdir, name + ".o"), []))
    for src, obj, defs in units:
        subprocess.check_call(base + defs + ["-c", src, "-o", obj])
    subprocess.check_call([nvcc, *ARCH, "-shared", "-o", SO + ".tmp"] + [o for _, o, _ in units])
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    print(build_lib(force=True, verbose=True))
