"""Build libdgz.so in-tree: nvcc for sm_100a only (no PTX fallback, no other arch).

    python -m paper_2103_03330_b200.build [--force]

Writes ``paper_2103_03330_b200/libdgz.so`` and ``build/ptxas.log`` (registers / spills per
kernel from ``-Xptxas -v``).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
SO = os.path.join(PKG, "libdgz.so")
BUILD = os.path.join(ROOT, "build", "dgz")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-Xptxas", "-v", "-I", INC, "-I", CSRC]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _stale(deps, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(INC, "dgz.h")] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".h")]
    srcs = sources()
    objs = [os.path.join(BUILD, os.path.basename(s)[:-3] + ".o") for s in srcs]
    todo = [(s, o) for s, o in zip(srcs, objs) if force or _stale([s] + headers, o)]

    def compile_one(so):
        s, o = so
        cmd = [NVCC, *ARCH, *FLAGS, "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stdout}\n{r.stderr}")
        return s, r.stderr

    logs = []
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            for s, err in ex.map(compile_one, todo):
                logs.append(f"==== {os.path.basename(s)}\n{err}")
        with open(os.path.join(ROOT, "build", "ptxas.log"), "a") as f:
            f.write("\n".join(logs))
    if force or todo or _stale(objs, SO):
        tmp = SO + f".tmp{os.getpid()}"
        cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-Xcompiler", "-fPIC", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, SO)
    # a plain C program against the C ABI (examples/c_abi_gather.c): proves the boundary needs
    # nothing but include/dgz.h, libdgz.so and the CUDA runtime
    ex_src = os.path.join(ROOT, "examples", "c_abi_gather.c")
    ex_bin = os.path.join(ROOT, "examples", "c_abi_gather")
    if os.path.exists(ex_src) and (force or _stale([ex_src, SO, os.path.join(INC, "dgz.h")], ex_bin)):
        cmd = ["gcc", "-O2", "-std=c11", "-I", INC, "-I", "/usr/local/cuda/include", ex_src, "-o", ex_bin,
               "-L", PKG, "-ldgz", "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,$ORIGIN/../paper_2103_03330_b200",
               "-Wl,-rpath,/usr/local/cuda/lib64"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"example build failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print("\n".join(logs))
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
