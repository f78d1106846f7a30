"""Build liblc.so (sm_100a) in-tree with nvcc. No JIT cache: the .so travels with the repo."""
import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "liblc.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              # fp64 geometry must round exactly like the oracle: no FMA contraction
              "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared"]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + [os.path.join(ROOT, "include", "lc.h")]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources() + headers())


def build(force=False, verbose=False):
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    inc = "-I" + os.path.join(ROOT, "include")
    odir = os.path.join(PKG, "build")
    os.makedirs(odir, exist_ok=True)
    comp = [f for f in NVCC_FLAGS if f != "-shared"]
    objs = []
    cmds = []
    for src in sources():   # one translation unit per kernel file, compiled in parallel
        obj = os.path.join(odir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        cmds.append([nvcc, *comp, inc, "-c", "-o", obj, src])
    if verbose:
        for cmd in cmds:
            print(" ".join(cmd))
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 4)) as ex:
        list(ex.map(subprocess.check_call, cmds))
    link = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs]
    if verbose:
        print(" ".join(link))
    subprocess.check_call(link)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
