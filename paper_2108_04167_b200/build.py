"""Build libsvmhss.so in-tree with nvcc for sm_100a (no torch types, plain C-ABI).

python paper_2108_04167_b200/build.py [--force]   (also called by __graft_entry__.build())
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsvmhss.so")
SOURCES = ["dense.cu", "cpqr.cu", "sort.cu", "tiles.cu", "tree.cu", "hss.cu", "ulv.cu", "admm.cu", "comm.cu", "shard.cu", "ann.cu", "api.cu"]
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _nccl_include():
    """The NCCL >= 2.28 headers with the device API (nccl_device.h), from the nvidia-nccl wheel
    torch ships with; None if absent (comm.cu then builds without the N3 device exchange)."""
    try:
        import nvidia.nccl as nn
        for base in list(getattr(nn, "__path__", [])):
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl_device.h")):
                return inc
    except ImportError:
        pass
    return None


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    extra = []
    if src == "comm.cu":
        inc = _nccl_include()
        if inc:
            extra = ["-I", inc, "-DSVMHSS_HAVE_NCCL_DEVICE"]
    cmd = [NVCC, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stderr}")
    return obj, p.stderr


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(HERE, "..", "include", "svmhss.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        res = list(ex.map(_compile, SOURCES))
    logs = "\n".join(r[1] for r in res)
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        f.write(logs)
    if verbose:
        print(logs)
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", LIB + ".tmp",
           *[r[0] for r in res], "-ldl"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"link failed:\n{p.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
