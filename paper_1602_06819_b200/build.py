"""Build libknng.so in-tree: nvcc for sm_100a (tcgen05-capable target), -lineinfo for ncu."""
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))
HDR = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + glob.glob(os.path.join(HERE, "csrc", "*.h")) +
             [os.path.join(HERE, "..", "include", "knng.h")])
OUT = os.environ.get("KNNG_BUILD_OUT") or os.path.join(HERE, "libknng.so")
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-shared"]


def stale():
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    return any(os.path.getmtime(f) > t for f in SRC + HDR)


def build(force=False, verbose=False):
    """Compile every .cu to an object in parallel (one nvcc per file), then link the shared library."""
    if not force and not stale():
        return OUT
    from concurrent.futures import ThreadPoolExecutor
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    cflags = [f for f in NVCC_FLAGS if f != "-shared"]
    if os.environ.get("KNNG_BUILD_PROFILE"):   # K1 cycle counters (KNNG_PROFILE=1 at run time)
        cflags.append("-DKNNG_PROFILE_COUNTERS")
    if os.environ.get("KNNG_BUILD_FLAGS"):   # extra nvcc flags (measurement variants, e.g. -DKNNG_K1_MB=8)
        cflags += os.environ["KNNG_BUILD_FLAGS"].split()
    if os.environ.get("KNNG_BUILD_HACK"):   # timing experiments only (wrong results): see knng_search.cu
        cflags.append("-DKNNG_HACK_" + os.environ["KNNG_BUILD_HACK"])
    if os.environ.get("KNNG_BUILD_DEBUG_WAIT"):   # K1 ring waits report a stuck producer / consumer
        cflags.append("-DKNNG_DEBUG_WAIT")
    jobs = []
    for src in SRC:
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".%d.o" % os.getpid())
        jobs.append((["nvcc"] + cflags + ["-c", src, "-o", obj], obj))
    if verbose:
        for cmd, _ in jobs:
            print(" ".join(cmd), file=sys.stderr)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        rcs = list(ex.map(lambda j: subprocess.run(j[0]).returncode, jobs))
    if any(rcs):
        for _, obj in jobs:
            if os.path.exists(obj):
                os.remove(obj)
        raise subprocess.CalledProcessError(max(rcs), "nvcc")
    tmp = OUT + ".tmp%d" % os.getpid()
    link = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp] + [o for _, o in jobs]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.check_call(link)
    for _, obj in jobs:
        os.remove(obj)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
