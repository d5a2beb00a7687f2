"""Builds the sm_100a C-ABI library in-tree: paper_2510_21956_b200/libla_cuda.so.

nvcc only (no torch extension machinery): the product is a plain C-ABI shared
library over include/la_cuda.h. Objects are cached under build/ and rebuilt
when a source or header is newer.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libla_cuda.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v" if os.environ.get("LA_PTXAS_VERBOSE") else "-O3"]
if os.environ.get("LA_TRACE"):  # clock64 pipeline traces (diagnostics, la_internal_trace_read*)
    FLAGS.append("-DLA_TRACE")
    if os.environ.get("LA_TRACE_G"):
        FLAGS.append("-DLA_TRACE_G=" + os.environ["LA_TRACE_G"])


def build_id() -> str:
    """git revision of the sources (+ "-dirty" with local edits) and the UTC build time."""
    import datetime
    try:
        rev = subprocess.run(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"], capture_output=True,
                             text=True, check=True).stdout.strip()
        dirty = subprocess.run(["git", "-C", ROOT, "status", "--porcelain", "--", "paper_2510_21956_b200/csrc",
                                "include"], capture_output=True, text=True).stdout.strip()
        rev += "-dirty" if dirty else ""
    except Exception:
        rev = "nogit"
    return rev + " " + datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%MZ")


def _newest(paths):
    return max(os.path.getmtime(p) for p in paths)


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    hdr_time = _newest(headers)
    objs = []
    for src in sources:
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        objs.append(obj)
        if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_time):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < _newest(objs):
        # build provenance (la_version): one C object with the revision and link time
        stamp_c, stamp_o = os.path.join(ROOT, "build", "la_build_id.c"), os.path.join(OBJ, "la_build_id.o")
        with open(stamp_c, "w") as f:
            f.write(f'const char la_build_id_str[] = "{build_id()}";\n')
        subprocess.run(["gcc", "-c", "-fPIC", "-o", stamp_o, stamp_c], check=True)
        objs = objs + [stamp_o]
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "shared",
               "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
