"""Build libknng.so in-tree: nvcc for sm_100a (tcgen05-capable target), -lineinfo for ncu."""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HDR = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(os.path.join(HERE, "csrc", "*.h")) +
             [os.path.join(HERE, "..", "include", "knng.h")])
OUT = os.path.join(HERE, "libknng.so")
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared"]


def stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(f) > t for f in SRC + HDR)


def build(force=False, verbose=False):
    if not force and not stale():
        return OUT
    tmp = OUT + ".tmp%d" % os.getpid()
    cmd = ["nvcc"] + NVCC_FLAGS + ["-o", tmp] + SRC
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
