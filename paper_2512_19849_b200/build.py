"""Build libepb200.so (the C-ABI boundary, include/epb.h) in-tree with nvcc.

All CUDA sources are compiled for sm_100a only (``-gencode
arch=compute_100a,code=sm_100a``) with ``-lineinfo`` so ncu's source page maps
to the kernels.  The CUDA runtime is linked statically so the library does not
depend on which libcudart torch loaded.  The output lands next to this file,
which is where ``_lib.py`` loads it from (and what gpurun ships to the box).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libepb200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-Wall", f"-I{ROOT / 'include'}",
          "-Wno-deprecated-gpu-targets"]
CU_FLAGS = ARCH + COMMON + ["--expt-relaxed-constexpr", "-Xptxas", "-O3"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA extension cannot be built")


def _sources():
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cpp"))


def _headers():
    return list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list((ROOT / "include").glob("*.h"))


def build(force: bool = False, verbose: bool = False, ptxas_verbose: bool = False) -> Path:
    nvcc = _nvcc()
    OBJ.mkdir(parents=True, exist_ok=True)
    hdr_mtime = max((h.stat().st_mtime for h in _headers()), default=0.0)
    objs = []
    for src in _sources():
        obj = OBJ / (src.name + ".o")
        objs.append(obj)
        stale = force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr_mtime)
        if not stale:
            continue
        flags = list(CU_FLAGS) if src.suffix == ".cu" else list(COMMON)
        if ptxas_verbose and src.suffix == ".cu":
            flags += ["-Xptxas", "-v"]
        cmd = [nvcc, "-c", str(src), "-o", str(obj)] + flags
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    lib_stale = force or not LIB.exists() or any(o.stat().st_mtime > LIB.stat().st_mtime for o in objs)
    if lib_stale:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [nvcc, "-shared", "-o", str(tmp)] + [str(o) for o in objs] + ARCH + [
            "-cudart", "static", "-Xcompiler", "-fPIC", "-Xlinker", "-soname=libepb200.so", "-lpthread", "-ldl",
            "-lrt"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB)
    build_ext(force=force or lib_stale, verbose=verbose)
    return LIB


EXT = PKG / "_epb_ext.so"


def build_ext(force: bool = False, verbose: bool = False) -> Path:
    """The C++ per-call host runtime (pybind11 + ATen), a client of libepb200.so.
    It resolves libepb200.so by SONAME; _lib.py loads that library first."""
    src = CSRC / "ext" / "epb_ext.cpp"
    deps = [src, LIB, ROOT / "include" / "epb.h"]
    if not force and EXT.exists() and EXT.stat().st_mtime >= max(d.stat().st_mtime for d in deps):
        return EXT
    from torch.utils.cpp_extension import load
    bdir = ROOT / "build" / "ext"
    bdir.mkdir(parents=True, exist_ok=True)
    import ctypes
    ctypes.CDLL(str(LIB), mode=os.RTLD_NOW | ctypes.RTLD_GLOBAL)  # so the import inside load() resolves it
    load(name="_epb_ext", sources=[str(src)], extra_include_paths=[str(ROOT / "include")],
         extra_cflags=["-O3", "-std=c++17"], extra_ldflags=[f"-L{PKG}", "-l:libepb200.so"],
         build_directory=str(bdir), with_cuda=True, verbose=verbose, is_python_module=True)
    tmp = EXT.with_suffix(".so.tmp")
    shutil.copy(bdir / "_epb_ext.so", tmp)
    os.replace(tmp, EXT)
    return EXT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, ptxas_verbose="-v" in sys.argv)
    print(LIB)
