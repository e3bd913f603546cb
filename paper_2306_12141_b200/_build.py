"""Build librecoil.so in-tree: host C++ (g++) + CUDA kernels for sm_100a (nvcc).

``python -m paper_2306_12141_b200._build`` or ``__graft_entry__.build()``.
The .so is git-ignored but travels to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "librecoil.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_INC = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include")
CXXFLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-Wno-unused-parameter", f"-I{INCLUDE}", f"-I{CUDA_INC}"]
NVFLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", f"-I{INCLUDE}", "-Xptxas", "-v"]


def _sources():
    host = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    cuda = sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(INCLUDE, "*.h")))
    return host, cuda, headers


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    host, cuda, headers = _sources()
    os.makedirs(BUILD, exist_ok=True)
    objs = []
    for src in host:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if force or _stale(obj, [src] + headers):
            subprocess.check_call(["g++", *CXXFLAGS, "-c", src, "-o", obj])
        objs.append(obj)
    for src in cuda:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        if force or _stale(obj, [src] + headers):
            res = subprocess.run([NVCC, *NVFLAGS, "-c", src, "-o", obj], capture_output=True, text=True)
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            with open(os.path.join(BUILD, os.path.basename(src) + ".ptxas.txt"), "w") as fh:
                fh.write(res.stderr)
            if verbose:
                sys.stderr.write(res.stderr)
        objs.append(obj)
    if force or _stale(LIB, objs):
        subprocess.check_call([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lpthread", "-ldl"])
    return LIB


def build_c_client() -> str:
    """examples/c_client.c: the C ABI from plain C (gcc, linked against librecoil.so and cudart)."""
    build()
    src = os.path.join(ROOT, "examples", "c_client.c")
    exe = os.path.join(ROOT, "examples", "c_client")
    if _stale(exe, [src, LIB, os.path.join(INCLUDE, "recoil.h")]):
        cuda_lib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", f"-I{INCLUDE}", f"-I{CUDA_INC}", src,
                               "-o", exe, f"-L{PKG}", "-lrecoil", f"-Wl,-rpath,{PKG}", f"-L{cuda_lib}", "-lcudart",
                               f"-Wl,-rpath,{cuda_lib}"])
    return exe


def build_sanitized() -> str:
    """Host library objects with ASan + UBSan (SURVEY §4 "Sanitizers"), linked with the regular
    CUDA kernel objects into librecoil_san.so (tools/sanitize_host.sh loads it through RECOIL_LIB)."""
    build()
    host, cuda, headers = _sources()
    out_dir = os.path.join(PKG, "build_san")
    os.makedirs(out_dir, exist_ok=True)
    san = ["-fsanitize=address,undefined", "-fno-omit-frame-pointer", "-fno-sanitize-recover=undefined", "-O1", "-g"]
    objs = []
    for src in host:
        obj = os.path.join(out_dir, os.path.basename(src) + ".o")
        if _stale(obj, [src] + headers):
            subprocess.check_call(["g++", *CXXFLAGS, *san, "-c", src, "-o", obj])
        objs.append(obj)
    objs += [os.path.join(BUILD, os.path.basename(src) + ".o") for src in cuda]
    lib = os.path.join(PKG, "librecoil_san.so")
    cuda_lib = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")
    subprocess.check_call(["g++", "-shared", *san, "-o", lib, *objs, f"-L{cuda_lib}", "-lcudart", "-lpthread", "-ldl",
                           f"-Wl,-rpath,{cuda_lib}"])
    return lib


if __name__ == "__main__":
    if "--sanitize" in sys.argv:
        print(build_sanitized())
    else:
        print(build(force="--force" in sys.argv, verbose=True))
