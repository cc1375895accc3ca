"""Builds the in-tree C-ABI library ``libqsim.so`` for sm_100a with nvcc.

    python -m paper_1802_06952_b200.build [--verbose]

Every .cu under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked (static cudart,
system NCCL) into ``paper_1802_06952_b200/libqsim.so``.  Rebuilds only when a source
or header is newer than the library.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libqsim.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# NCCL: the copy bundled with torch (same SONAME libnccl.so.2 as the one torch loads, so the
# process holds a single NCCL whichever of torch / libqsim is loaded first)
try:
    import nvidia.nccl as _nccl
    NCCL_DIR = os.path.dirname(_nccl.__file__) if _nccl.__file__ else list(_nccl.__path__)[0]
except Exception:  # fall back to the system NCCL
    NCCL_DIR = None
NCCL_INC = os.path.join(NCCL_DIR, "include") if NCCL_DIR else "/usr/include"
NCCL_LIB = os.path.join(NCCL_DIR, "lib") if NCCL_DIR else "/usr/lib/x86_64-linux-gnu"
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-I", NCCL_INC, "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cpp")) + \
        [os.path.join(ROOT, "include", "qsim.h"), __file__]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")))

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, "-x", "cu", *ARCH, *FLAGS, "-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources() + cpp))
    tmp = LIB + ".tmp"
    nccl_so = os.path.join(NCCL_LIB, "libnccl.so.2")
    link_nccl = ["-L", NCCL_LIB, "-Xlinker", "-l:libnccl.so.2"] if os.path.exists(nccl_so) else ["-lnccl"]
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, *link_nccl, "-Xlinker", f"-rpath={NCCL_LIB}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
