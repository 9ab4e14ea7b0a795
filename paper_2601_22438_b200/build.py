"""Build libkvring.so in-tree for sm_100a (nvcc + g++, static cudart).

``python -m paper_2601_22438_b200.build`` or ``__graft_entry__.build()``.
The shared object lands next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libkvring.so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES_CU = ["kvring_kernels.cu", "kvring_step.cu"]
SOURCES_CPP = ["kvring_host.cpp"]
HEADERS = ["kvring_internal.h"]


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "kvring.h")]
    objs = []
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            cmd = [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xcompiler", "-fvisibility=hidden", "-I", INCLUDE, "-I", CSRC,
                   "-c", s, "-o", o]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
            extra = os.environ.get("KVRING_NVCC_DEFS", "")   # debug builds: -DKV_BOUNDS_CHECK
            if extra:
                cmd[1:1] = extra.split()
            _run(cmd)
        objs.append(o)
    for src in SOURCES_CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs):
            _run(["g++", "-O2", "-g", "-std=c++17", "-fPIC", "-fvisibility=hidden", "-Wall",
                  "-I", INCLUDE, "-I", CSRC, "-I", os.path.join(CUDA_HOME, "include"),
                  "-c", s, "-o", o])
        objs.append(o)
    if force or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        _run([NVCC, *ARCH, "-shared", "-cudart=static", "-Xcompiler", "-fPIC", "-o", tmp, *objs,
              "-lpthread"])
        shutil.move(tmp, LIB)
    return LIB


NCCL_HOME = None
try:  # the NCCL that ships with the torch venv (2.28; not the system /usr/include copy)
    import nvidia.nccl as _nv_nccl
    NCCL_HOME = list(_nv_nccl.__path__)[0]
except Exception:
    pass
LIB_NCCL = os.path.join(HERE, "libkvnccl.so")


def build_nccl(force: bool = False) -> str | None:
    """libkvnccl.so: the NCCL comparison transport's native driver (a6)."""
    if NCCL_HOME is None:
        return None
    src = os.path.join(CSRC, "kvnccl.cpp")
    deps = [src, os.path.join(INCLUDE, "kvnccl.h")]
    if force or _stale(LIB_NCCL, deps):
        lib = os.path.join(NCCL_HOME, "lib")
        tmp = LIB_NCCL + ".tmp"
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-fvisibility=hidden", "-Wall",
              "-I", INCLUDE, "-I", os.path.join(NCCL_HOME, "include"),
              "-I", os.path.join(CUDA_HOME, "include"), src, "-o", tmp,
              "-L", lib, "-l:libnccl.so.2", f"-Wl,-rpath,{lib}",
              "-L", os.path.join(CUDA_HOME, "lib64"), "-lcudart"])
        shutil.move(tmp, LIB_NCCL)
    return LIB_NCCL


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
    build_nccl(force="--force" in sys.argv)
