"""Build the in-tree CUDA library libdynamoe_b200.so for sm_100a with nvcc.

Each .cu under csrc/ is compiled to an object (in parallel) and linked into one shared
library that exports the C ABI declared in include/moe.h.  No torch headers are used.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libdynamoe_b200.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def nccl_include():
    """Headers of the NCCL torch loads (nccl.h + the NCCL >= 2.28 device API, nccl_device.h):
    the nvidia-nccl wheel in this environment; only the peer-window path (nccl_lsa.cu) uses
    them, and the library itself is resolved at run time (dlopen)."""
    try:
        import nvidia
        for base in nvidia.__path__:
            inc = os.path.join(base, "nccl", "include")
            if os.path.exists(os.path.join(inc, "nccl_device.h")):
                return inc
    except ImportError:
        pass
    raise RuntimeError("nccl_device.h (NCCL >= 2.28 headers, nvidia-nccl wheel) not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _needs(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "moe.h"))
    srcs = sources()
    objs = []
    jobs = []
    for src in srcs:
        obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _needs(obj, [src] + headers):
            cmd = [NVCC, *ARCH, *FLAGS, *os.environ.get("MOE_NVCC_EXTRA", "").split(), "-c", src,
                   "-o", obj]
            if os.path.basename(src) == "nccl_lsa.cu":
                cmd[1:1] = ["-I", nccl_include()]
            if os.environ.get("MOE_PTXAS_V"):
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, r in ex.map(run, jobs):
            if verbose or r.returncode != 0 or os.environ.get("MOE_PTXAS_V"):
                sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {cmd[-3]}")
    if force or jobs or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
