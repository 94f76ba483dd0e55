"""Builds libchm.so in-tree: nvcc for sm_100a (CUDA kernels) + g++ flags for the host runtime.

    python -m paper_2509_11076_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libchm.so")
LIB_DEBUG = os.path.join(HERE, "libchm_debug.so")  # device-side bounds checks (CHM_DEBUG)
SOURCES = ["core.cpp", "trace.cpp", "executor.cpp", "generator.cpp", "oom.cpp", "trace_io.cpp", "stall.cpp", "arena.cpp", "swap.cu", "replay.cu", "timeline.cu", "explicit.cu", "descend.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, "internal.h"), os.path.join(CSRC, "eval_common.cuh"),
                                                       os.path.join(ROOT, "include", "chm.h"),
                                                       os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    """debug: libchm_debug.so with device-side bounds checks (CHM_DCHECK -> trap); load it with
    CHM_LIB=<path> to run the tests against it"""
    lib = LIB_DEBUG if debug else LIB
    if not force and not _stale(lib):
        return lib
    objdir = os.path.join(HERE, "build_debug" if debug else "build")
    os.makedirs(objdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-I", os.path.join(ROOT, "include"),
              "-Xcompiler", "-fPIC,-ffp-contract=off,-Wall", "--fmad=false"] + ARCH + (["-DCHM_DEBUG"] if debug else [])
    objs = []
    for src in SOURCES:
        obj = os.path.join(objdir, src + ".o")
        cmd = [NVCC] + common + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd += ["-x", "cu"] if False else []
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs +
                          ["-Xlinker", "-rpath,/usr/local/cuda/lib64", "-lcudart_static", "-lrt", "-lpthread", "-ldl"])
    os.replace(tmp, lib)
    return lib


HOOK_DIR = os.path.join(HERE, "build_hook")
HOOK_SRC = os.path.join(CSRC, "hook.cpp")
HOOK_NAME = "chm_hook"


def hook_path() -> str:
    return os.path.join(HOOK_DIR, HOOK_NAME + ".so")


def build_hook(force: bool = False, verbose: bool = False) -> str:
    """the profiler hook at operator dispatch (csrc/hook.cpp): a PyTorch C++ extension, built
    in-tree (build_hook/chm_hook.so) with torch's own compiler flags; it calls libchm through the
    addresses of its C entry points, so it does not link it"""
    so = hook_path()
    deps = [HOOK_SRC, os.path.join(ROOT, "include", "chm.h"), os.path.abspath(__file__)]
    if not force and os.path.exists(so) and all(os.path.getmtime(d) <= os.path.getmtime(so) for d in deps):
        return so
    os.makedirs(HOOK_DIR, exist_ok=True)
    from torch.utils import cpp_extension
    cpp_extension.load(name=HOOK_NAME, sources=[HOOK_SRC], build_directory=HOOK_DIR,
                       extra_include_paths=[os.path.join(ROOT, "include"), "/usr/local/cuda/include"],
                       extra_cflags=["-O3", "-std=c++17"], extra_ldflags=["-lc10_cuda"], with_cuda=False,
                       is_python_module=True, verbose=verbose)
    os.utime(so)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
    if "--no-hook" not in sys.argv:
        print(build_hook(force="--force" in sys.argv, verbose="-v" in sys.argv))
