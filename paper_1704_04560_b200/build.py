"""Builds libmtx.so (the C-ABI of include/mtx.h) for sm_100a with nvcc, in-tree.

Every .cu under csrc/ is compiled with
    -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17
(SASS embedded for B200; no PTX JIT needed on the box), against the NCCL that
PyTorch ships (one libnccl per process), with the CUDA runtime linked
statically.  Objects are cached by source/header mtime.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libmtx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _flags(inc):
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
                   "-I", inc, "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"] + \
        (["-DMTX_TRACE=1"] if os.environ.get("MTX_TRACE") == "1" else []) + \
        (["-DMTX_TC_EXPERIMENTS=1"] if os.environ.get("MTX_TC_EXPERIMENTS") == "1" else [])  # dev builds (force=True)


def build(force: bool = False, verbose: bool = False) -> str:
    inc, libdir = nccl_dirs()
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "mtx.h")])
    dep_mtime = max(os.path.getmtime(d) for d in deps)
    objs, todo = [], []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), dep_mtime):
            todo.append((s, o))

    def compile_one(so):
        s, o = so
        cmd = [NVCC, *_flags(inc), "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(o + ".log", "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        return s, r

    # the translation units are independent: compile them concurrently
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        results = list(ex.map(compile_one, todo))
    for s, r in results:
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            print(r.stderr)
    rebuilt = bool(todo)
    if rebuilt or force or not os.path.exists(LIB):
        tmp = LIB + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L", libdir, "-l:libnccl.so.2",
               "-Xlinker", f"-rpath={libdir}", "-lcuda" if False else ""]
        cmd = [c for c in cmd if c]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
