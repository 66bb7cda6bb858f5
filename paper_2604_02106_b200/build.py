"""Build libhgrd_gpu.so in-tree for sm_100a (nvcc + the system g++).

The library holds the host front end (csrc/host: MiniCU parser, host
interpreter mirror, kernel lowering), the C ABI (csrc/capi.cpp) and the
CUDA race-check stage (csrc/gpu).  Objects go to build/ (git-ignored);
the .so lands next to this file so it travels to the GPU box with the repo.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "hgrd_gpu")
LIB = os.path.join(HERE, "libhgrd_gpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = ["-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(CSRC, "host")]


def _sources():
    out = []
    for sub in ("host", "gpu", ""):
        d = os.path.join(CSRC, sub)
        for f in sorted(os.listdir(d)):
            p = os.path.join(d, f)
            if os.path.isfile(p) and f.endswith((".cpp", ".cu")):
                out.append(p)
    return out


def _headers():
    inc = os.path.join(ROOT, "include")
    hs = [os.path.join(inc, f) for f in os.listdir(inc) if f.endswith(".h")]
    for sub in ("host", "gpu", ""):
        d = os.path.join(CSRC, sub)
        hs += [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".hpp", ".cuh"))]
    return hs


def _compile(src: str) -> str:
    obj = os.path.join(BUILD, os.path.relpath(src, CSRC).replace(os.sep, "_") + ".o")
    newest = max(os.path.getmtime(h) for h in _headers() + [src, __file__])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest:
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC, *ARCH, "-O3", "-std=c++17", "-lineinfo", "--extended-lambda",
               "-Xcompiler", "-fPIC", "-Xptxas", "-v", *INCLUDES, "-c", src, "-o", obj]
    else:
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-Wall", "-Wextra", *INCLUDES,
               "-I/usr/local/cuda/include", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if src.endswith(".cu"):
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(_compile, srcs))
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs,
               "-Xlinker", "--exclude-libs,ALL", "-lpthread", "-ldl",
               "-L/usr/local/cuda/lib64", "-lnvrtc", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
