"""Builds an A/B variant of libchm.so with extra nvcc defines for one source (default replay.cu),
linking the other objects from the regular build: paper_2509_11076_b200/libchm_<name>.so (git-
ignored; load it with CHM_LIB=<path>, e.g. under tools/eval_time.py).

    python tools/build_variant.py <name> [-DFOO=1 ...] [--src replay.cu]"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_11076_b200 import build as B  # noqa: E402


def main():
    name = sys.argv[1]
    defs = [a for a in sys.argv[2:] if a.startswith("-D")]
    src = sys.argv[sys.argv.index("--src") + 1] if "--src" in sys.argv else "replay.cu"
    B.build()
    objdir = os.path.join(B.HERE, "build")
    vdir = os.path.join(B.HERE, f"build_var_{name}")
    os.makedirs(vdir, exist_ok=True)
    common = ["-O3", "-std=c++17", "-lineinfo", "-I", os.path.join(B.ROOT, "include"),
              "-Xcompiler", "-fPIC,-ffp-contract=off,-Wall", "--fmad=false"] + B.ARCH
    vobj = os.path.join(vdir, src + ".o")
    subprocess.check_call([B.NVCC] + common + defs + ["-Xptxas", "-v", "-c", os.path.join(B.CSRC, src), "-o", vobj])
    objs = [vobj if s == src else os.path.join(objdir, s + ".o") for s in B.SOURCES]
    lib = os.path.join(B.HERE, f"libchm_{name}.so")
    subprocess.check_call([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + objs +
                          ["-Xlinker", "-rpath,/usr/local/cuda/lib64", "-lcudart_static", "-lrt", "-lpthread", "-ldl"])
    print(lib)


if __name__ == "__main__":
    main()
