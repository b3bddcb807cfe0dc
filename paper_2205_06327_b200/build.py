"""Build libptycho.so (sm_100a) in-tree with nvcc.  No JIT cache: the .so travels with the repo."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libptycho.so")
DEBUG_LIB = os.path.join(LIBDIR, "libptycho_debug.so")
SOURCES = ["kernels.cu", "api.cu"]
HEADERS = ["internal.h", "twiddle32.h"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        inc = os.path.join(base, "nccl", "include")
        lib = os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("NCCL headers not found (expected nvidia/nccl in site-packages)")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "ptycho.h")]
    if not os.path.exists(DEMO) or os.path.getmtime(DEMO_SRC) > os.path.getmtime(DEMO):
        return True
    if not os.path.exists(DEBUG_LIB) or os.path.getmtime(DEBUG_LIB) < t:
        return True
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(defines, out, verbose):
    """Start nvcc for every source of one library variant; returns (processes, objects, link cmd)."""
    inc, libdir = nccl_dirs()
    nvcc = os.environ.get("NVCC", "nvcc")
    common = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", inc]
    common += ["-D" + d for d in defines]
    tag = "" if out == LIB else "_" + os.path.basename(out).replace(".so", "")
    objs, procs = [], []
    for src in SOURCES:
        obj = os.path.join(LIBDIR, src.replace(".cu", tag + ".o"))
        cmd = [nvcc] + common + ["-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    link = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", out] + objs + \
        ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + libdir, "--cudart", "static"]
    return procs, link


def build(force: bool = False, verbose: bool = True, defines=(), out=None) -> str:
    """defines / out: experimental variants (e.g. ["PTYCHO_MIN2"], "lib/libptycho_a.so").  The
    default build makes the product library and, compiled concurrently, the ordering-check variant
    lib/libptycho_debug.so (-DPTYCHO_DEBUG_CHECKS; ptycho_debug_errors, tests/test_gpu_ordering.py)."""
    lib_out = out or LIB
    if out is None and not force and not _stale():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    variants = [(list(defines), lib_out)]
    if out is None:
        variants.append((list(defines) + ["PTYCHO_DEBUG_CHECKS"], DEBUG_LIB))
    jobs = [_compile(d, o, verbose) for d, o in variants]
    for procs, _ in jobs:
        for p in procs:
            if p.wait() != 0:
                raise RuntimeError("nvcc failed")
    for _, link in jobs:
        if verbose:
            print(" ".join(link), flush=True)
        subprocess.check_call(link)
    if out is None:
        build_demo(verbose)
    return lib_out


DEMO_SRC = os.path.join(ROOT, "examples", "ptycho_demo.c")
DEMO = os.path.join(LIBDIR, "ptycho_demo")


def build_demo(verbose: bool = True) -> str:
    """examples/ptycho_demo.c: plain C against include/ptycho.h + libptycho.so (no Python)."""
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
           DEMO_SRC, "-o", DEMO, "-L", LIBDIR, "-lptycho", "-Wl,-rpath," + LIBDIR,
           "-L", os.path.join(cuda, "lib64"), "-lcudart", "-Wl,-rpath," + os.path.join(cuda, "lib64"), "-lm"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    return DEMO


if __name__ == "__main__":
    build(force="--force" in sys.argv)
