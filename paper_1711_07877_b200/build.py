"""Build the in-tree native library paper_1711_07877_b200/libsbd_b200.so.

nvcc compiles the sm_100a kernels (``-gencode arch=compute_100a,code=sm_100a
-lineinfo``), g++ the host C++; the result links cuFFT and a static CUDA
runtime. Run ``python paper_1711_07877_b200/build.py`` (as a script: importing the package
needs the built library) or call ``build()``.
Cross-compiles on a machine without a GPU.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsbd_b200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["kernels.cu", "assemble_kernels.cu"]
CPP_SOURCES = ["window.cpp", "plan.cpp", "op.cpp", "slab.cpp", "assemble.cpp", "bessel_host.cpp", "sbd_fit.cpp"]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")
    elif verbose and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "sbd_b200.h"))
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            _run([NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-v" if verbose else "-O3", "-c", s, "-o", o], verbose)
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            _run(["g++", "-std=gnu++17", "-O2", "-fPIC", "-fopenmp", "-Wall", "-Wno-unused-function",
                  f"-I{CUDA}/include", "-c", s, "-o", o], verbose)
    if force or _stale(LIB, objs):
        tmp = LIB + ".tmp"
        _run(["g++", "-shared", "-o", tmp, *objs, f"-L{CUDA}/lib64", "-lcufft", "-lcusolver", "-lcudart_static", "-fopenmp",
              "-ldl", "-lrt", "-lpthread", f"-Wl,-rpath,{CUDA}/lib64"], verbose)
        shutil.move(tmp, LIB)
    # the C++ API example (include/sbd_b200.hpp) links the library like a user would
    ex_src = os.path.join(HERE, "..", "examples", "apply_example.cpp")
    ex_bin = os.path.join(OBJ, "apply_example")
    if os.path.exists(ex_src) and (force or _stale(ex_bin, [ex_src, LIB] + headers +
                                                   [os.path.join(HERE, "..", "include", "sbd_b200.hpp")])):
        _run(["g++", "-std=c++17", "-O2", f"-I{os.path.join(HERE, '..', 'include')}", ex_src, "-o", ex_bin,
              f"-L{HERE}", "-lsbd_b200", f"-Wl,-rpath,{HERE}"], verbose)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
