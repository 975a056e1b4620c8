"""Build libddg.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libddg.so")
SOURCES = ["pcg.cu", "symv.cu", "coarse.cu", "setup_kernels.cu", "chol.cu", "basis.cu", "setup.cpp", "coarse_sparse.cpp", "dist.cpp",
           "comm.cpp"]
HEADERS = ["ddg_internal.h", "kernel_common.cuh", "ctx.h", "dist.h", "comm.h", os.path.join("..", "..", "include", "ddg.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir():
    for p in sys.path + ["/opt/prime-rl/.venv/lib/python3.12/site-packages"]:
        cand = os.path.join(p, "nvidia", "nccl")
        if os.path.exists(os.path.join(cand, "include", "nccl.h")):
            return cand
    if os.path.exists("/usr/include/nccl.h"):
        return "/usr"
    raise RuntimeError("nccl.h not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    bdir = os.path.join(CSRC, "build")
    os.makedirs(bdir, exist_ok=True)

    def compile_one(s):
        src = os.path.join(CSRC, s)
        obj = os.path.join(bdir, s + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
               "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"),
               "-I", os.path.join(_nccl_dir(), "include"),
               f'-DDDG_NCCL_DIR="{os.path.join(_nccl_dir(), "lib")}"',
               "-c", src, "-o", obj]
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs,
                           "-lpthread", "-ldl"])
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose="-v" in sys.argv))
