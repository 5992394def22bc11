"""Build libhinm_b200.so (in-tree) with nvcc for sm_100a.

    python -m paper_2407_20496_b200.build                # incremental
    python -m paper_2407_20496_b200.build --force
    python -m paper_2407_20496_b200.build --experiments  # scripts/libhinm_b200_exp.so

The experiments library (-DHINM_EXPERIMENTS) adds timing-only SpMM variants whose results are
garbage (HINM_GATHER=dbg_*); it is used by scripts/ through HINM_B200_LIB and never by the package.

The shared library is plain C-ABI (include/hinm_b200.h); the Python package loads it with
ctypes.  Objects go to build/ (git-ignored); the .so lands next to this file so that it
travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libhinm_b200.so")
EXP_LIB = os.path.join(ROOT, "scripts", "libhinm_b200_exp.so")
SOURCES = ["compress.cu", "spmm_sm100.cu", "spmm_simt.cu", "chain_host.cu", "capi.cu",
           "icp.cu", "assignment.cu", "unpack.cu", "ocp.cu", "kmeans.cu", "group.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INCLUDE, "-I" + CSRC]
# experiments build only: extra defines (e.g. HINM_EXP_FLAGS="-DHINM_PAIR_STAGES=5")
EXP_FLAGS = os.environ.get("HINM_EXP_FLAGS", "").split()


def _deps_mtime() -> float:
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(INCLUDE, "hinm_b200.h"))
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, experiments: bool = False) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", "_exp.o" if experiments else ".o"))
    extra = ["-DHINM_EXPERIMENTS", *EXP_FLAGS] if experiments else []
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = True, experiments: bool = False) -> str:
    """Compile every CUDA source for sm_100a and link the in-tree shared library."""
    lib = EXP_LIB if experiments else LIB
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= _deps_mtime():
        return lib
    os.makedirs(BUILD, exist_ok=True)
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, experiments), SOURCES))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    if verbose:
        print(f"[hinm] built {lib}", file=sys.stderr)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--experiments", action="store_true")
    a = ap.parse_args()
    build(force=a.force, experiments=a.experiments)
