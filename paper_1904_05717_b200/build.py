"""Build the native library in-tree: paper_1904_05717_b200/lib/libtilemul_b200.so.

Host C++ (csrc/host/*.cpp, csrc/capi.cpp) with g++ -O2, kernels
(csrc/kernels/*.cu) with nvcc for sm_100a only, linked with the static CUDA
runtime so the .so carries no dependency on a particular libcudart.
Incremental: objects are rebuilt only when a source or header is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libtilemul_b200.so")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-std=c++17", "-O2", "-fPIC", "-Wall", "-Wno-unused-function", f"-I{CUDA_HOME}/include",
            f"-I{os.path.join(ROOT, 'include')}", f"-I{OBJ}"]
NVFLAGS = ARCH + ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                  f"-I{os.path.join(ROOT, 'include')}"] + os.environ.get("TILEMUL_B200_NVFLAGS", "").split()


def _headers():
    return glob.glob(os.path.join(CSRC, "**", "*.hpp"), recursive=True) + [
        os.path.join(ROOT, "include", "tilemul_b200.h")]


BUILD_ID = os.path.join(OBJ, "build_id.h")


def source_files():
    """Every file the library is built from (the build id hashes these)."""
    return sorted(glob.glob(os.path.join(CSRC, "**", "*.cpp"), recursive=True) +
                  glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True) +
                  glob.glob(os.path.join(CSRC, "**", "*.hpp"), recursive=True) +
                  [os.path.join(ROOT, "include", "tilemul_b200.h"), os.path.abspath(__file__)])


def kernel_files():
    """The sources that decide the device work of an execute() call: the
    kernels, the lowering onto CTA tasks, the host pipeline, the build flags."""
    return sorted(glob.glob(os.path.join(CSRC, "kernels", "*")) +
                  [os.path.join(CSRC, f) for f in ("lower.cpp", "engine.hpp", "host_pipe.cpp")] +
                  [os.path.abspath(__file__)])


def _hash(files) -> str:
    import hashlib

    h = hashlib.sha256()
    for f in files:
        h.update(os.path.relpath(f, ROOT).replace(os.sep, "/").encode() + b"\0")
        h.update(open(f, "rb").read())
    return h.hexdigest()[:16]


def source_hash() -> str:
    """sha256[:16] over all of the library's sources (paths relative to the
    repo, then contents): the build id compiled into the library
    (tm_build_id); the loader refuses a library built from other sources."""
    return _hash(source_files())


def kernel_hash() -> str:
    """sha256[:16] over kernel_files(): the kernel id (tm_kernel_id) stamped
    on every ncu summary, so a profile of other device code is detected."""
    return _hash(kernel_files())


def _write_build_id() -> None:
    text = (f'#pragma once\n#define TM_BUILD_ID "{source_hash()}"\n'
            f'#define TM_KERNEL_ID "{kernel_hash()}"\n')
    if not os.path.exists(BUILD_ID) or open(BUILD_ID).read() != text:
        with open(BUILD_ID, "w") as f:
            f.write(text)


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    obj = os.path.join(OBJ, rel + ".o")
    if not _stale(obj, [src] + _headers() + ([BUILD_ID] if src.endswith("capi.cpp") else [])):
        return obj, None
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + ["-c", src, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        return obj, f"$ {' '.join(cmd)}\n{r.stdout}{r.stderr}"
    return obj, None


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    if not os.path.exists(NVCC) and shutil.which("nvcc") is None:
        raise RuntimeError("nvcc not found; cannot build the sm_100a kernels")
    _write_build_id()
    srcs = sorted(glob.glob(os.path.join(CSRC, "**", "*.cpp"), recursive=True) +
                  glob.glob(os.path.join(CSRC, "**", "*.cu"), recursive=True))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        results = list(ex.map(_compile, srcs))
    errs = [e for _, e in results if e]
    if errs:
        raise RuntimeError("native build failed:\n" + "\n".join(errs))
    objs = [o for o, _ in results]
    if _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n$ {' '.join(cmd)}\n{r.stdout}{r.stderr}")
        if verbose:
            print("linked", LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
    sys.exit(0)
