"""Builds libtgk.so in-tree (paper_2602_05052_b200/lib/) for sm_100a.

nvcc cross-compiles here without a GPU; the .so travels to the GPU box with the
repo snapshot.  Device code is compiled with -fmad=false: the exact arithmetic
mode reproduces the reference's FMA-free operation order bit for bit (the fast
mode uses explicit __fma_rn intrinsics, which -fmad does not affect).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "lib")
OBJ = os.path.join(OUT, "obj")
LIB = os.path.join(OUT, "libtgk.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                  "-Xptxas", "-v", "--expt-relaxed-constexpr",
                  f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}"]
CXXFLAGS = ["-O3", "-fPIC", "-std=c++17", "-Wall", "-Wno-unused-function",
            f"-I{os.path.join(ROOT, 'include')}", f"-I{CSRC}", f"-I{os.path.join(CUDA, 'include')}"]

CU = ["routing.cu", "stage.cu", "fused.cu", "fast.cu", "batched.cu", "fused_elast.cu", "adjoint.cu", "solve.cu", "scatter.cu"]
CPP = ["host.cpp", "plan.cpp", "plan_entries.cpp", "plan_fast.cpp"]
HEADERS = ["tgk_internal.hpp", "element.cuh", "cuda_util.cuh"]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def _compile(src):
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    deps = [path] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "tgk.h")]
    if not _newer(deps, obj):
        return obj, ""
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + ["-c", path, "-o", obj]
    else:
        cmd = [os.environ.get("CXX", "g++")] + CXXFLAGS + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def variant(defines: list[str], name: str) -> str:
    """Experiment build with extra -D flags into lib/<name>.so (separate object dir)."""
    global OBJ, LIB, NVFLAGS
    saved = (OBJ, LIB, NVFLAGS)
    OBJ = os.path.join(OUT, "obj_" + name)
    LIB = os.path.join(OUT, name + ".so")
    NVFLAGS = NVFLAGS + [f"-D{d}" for d in defines]
    try:
        return build()
    finally:
        OBJ, LIB, NVFLAGS = saved


def build(verbose=False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with ThreadPoolExecutor(max_workers=8) as ex:
        results = list(ex.map(_compile, CU + CPP))
    objs = [o for o, _ in results]
    log = "\n".join(f"== {s}\n{msg}" for s, (_, msg) in zip(CU + CPP, results) if msg)
    if log:
        with open(os.path.join(OUT, "ptxas.log"), "w") as f:
            f.write(log)
    if verbose and log:
        print(log)
    if _newer(objs, LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", LIB] + objs + ["-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


def build_module() -> str:
    """The pybind11 module `_tgfem` (bindings/module.cpp: the reference's compiled
    Python module over the C ABI) into lib/, linked to libtgk.so by rpath."""
    import sysconfig

    import pybind11
    lib = build()
    src = os.path.join(HERE, "bindings", "module.cpp")
    out = os.path.join(OUT, "_tgfem" + sysconfig.get_config_var("EXT_SUFFIX"))
    if _newer([src, lib, os.path.join(ROOT, "include", "tgk.h")], out):
        cmd = [os.environ.get("CXX", "g++"), "-O2", "-shared", "-fPIC", "-std=c++17", "-fvisibility=hidden",
               f"-I{pybind11.get_include()}", f"-I{sysconfig.get_paths()['include']}", f"-I{os.path.join(ROOT, 'include')}",
               src, "-o", out, f"-L{OUT}", "-ltgk", "-Wl,-rpath,$ORIGIN"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"module build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    print(build_module())
