"""Build libbfapply.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2007_00202_b200.build
"""
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", f) for f in ("kernels.cu", "fast.cu", "leaf.cu", "plan.cu", "rmatvec.cu", "tile_umma.cu")]
LIB = os.path.join(PKG, "libbfapply.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills",
         "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(PKG, "csrc")]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = SRC + [os.path.join(PKG, "csrc", f) for f in os.listdir(os.path.join(PKG, "csrc"))]
    deps.append(os.path.join(ROOT, "include", "bfapply.h"))
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    extra = os.environ.get("BF_NVCC_EXTRA", "").split()  # experiments: e.g. -DBF_C64_NP=5
    cmd = [NVCC] + FLAGS + extra + SRC + ["-o", LIB + ".tmp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
