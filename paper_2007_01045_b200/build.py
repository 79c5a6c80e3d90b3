"""Builds libdapple.so in-tree (sm_100a only).

Host planner (C++20, -ffp-contract=off so the planner's doubles match the
reference bit for bit), CUDA stage kernels and the executor runtime
(nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo) are linked into one
shared library with a static CUDA runtime; NCCL is linked dynamically so the
process shares whatever libnccl.so.2 torch already loaded.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libdapple.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC]

CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall", "-Wextra", "-fvisibility=default"]
NVFLAGS = ARCH + ["-std=c++17", "-O3", "-lineinfo", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-ffp-contract=off"]


def _nccl_link():
    for d in ("/usr/lib/x86_64-linux-gnu", "/usr/lib64", "/usr/local/lib"):
        if os.path.exists(os.path.join(d, "libnccl.so")) or os.path.exists(os.path.join(d, "libnccl.so.2")):
            return ["-L" + d, "-l:libnccl.so.2"]
    raise RuntimeError("libnccl.so.2 not found")


def _sources():
    host = sorted(glob.glob(os.path.join(CSRC, "host", "*.cpp")))
    cuda = sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")) + glob.glob(os.path.join(CSRC, "*.cu")) +
                  glob.glob(os.path.join(CSRC, "runtime", "*.cu")))
    cpp_rt = sorted(glob.glob(os.path.join(CSRC, "runtime", "*.cpp")))
    return host, cuda, cpp_rt


def _headers_mtime():
    hs = glob.glob(os.path.join(CSRC, "**", "*.h*"), recursive=True) + \
        glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True) + \
        glob.glob(os.path.join(ROOT, "include", "**", "*.h*"), recursive=True)
    return max([os.path.getmtime(h) for h in hs] + [0.0])


def _obj_for(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "__")
    return os.path.join(BUILD, rel + ".o")


def _compile(src, hdr_mtime, verbose):
    obj = _obj_for(src)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + INCLUDES + ["-c", src, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + INCLUDES + ["-I" + os.path.join(CUDA, "include"), "-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
    return obj


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    if force:
        shutil.rmtree(BUILD)
        os.makedirs(BUILD)
    host, cuda, cpp_rt = _sources()
    hdr = _headers_mtime()
    with ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as pool:
        objs = list(pool.map(lambda s: _compile(s, hdr, verbose), host + cuda + cpp_rt))
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        tmp = LIB + ".tmp"
        cmd = ["g++", "-shared", "-o", tmp] + objs + [
            "-L" + os.path.join(CUDA, "lib64"), "-lcudart_static", "-lrt", "-lpthread", "-ldl"] + _nccl_link() + \
            ["-Wl,--no-undefined"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
