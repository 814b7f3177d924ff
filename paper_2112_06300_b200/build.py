"""In-tree build of the native libraries (sm_100a only).

    libccdk.so    CUDA kernels + the C ABI (include/ccdk.h)
    libccdkit.so  C++ host API with the reference signatures
                  (include/ccdkit/*.hpp) layered on libccdk.so
                  incl. the benchmark/audit layer (bench.hpp, OBJ ingestion)
    libccdkit_bench.so  end-to-end timing harness: ccdkit::ccd through
                  libccdkit.so from pageable host vectors (bench.py e2e)
    ccdbench      the audit/benchmark CLI over libccdkit.so (no oracle linked)

Both land in paper_2112_06300_b200/lib/ so they travel with the repository
snapshot to the GPU box.  Flags: no FMA contraction (--fmad=false, and the
kernels use explicit _rn intrinsics anyway), no fast-math, no FTZ.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
INCLUDE = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CU_SOURCES = ["ccdk_api.cu", "ccdk_geometry.cu", "ccdk_broad.cu", "ccdk_bfs.cu", "ccdk_distance.cu"]
CXX_SOURCES = ["ccdkit_host.cpp", "ccdkit_audit.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-warn-spills",
]


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout.strip() or r.stderr.strip()):
        print(r.stdout + r.stderr)
    return r


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_info: bool = False) -> str:
    os.makedirs(os.path.join(LIB, "obj"), exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h", ".hpp"))]
    headers.append(os.path.join(INCLUDE, "ccdk.h"))
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(LIB, "obj", src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            extra = ["-Xptxas", "-v"] if ptxas_info else []
            _run([NVCC, *NVCC_FLAGS, *extra, "-I", INCLUDE, "-I", CSRC, "-c", s, "-o", o], verbose)
    so = os.path.join(LIB, "libccdk.so")
    if force or _stale(so, objs):
        _run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", so,
              "-cudart", "static"], verbose)
    # C++ host API over the C ABI
    cxx = [os.path.join(CSRC, c) for c in CXX_SOURCES]
    so2 = os.path.join(LIB, "libccdkit.so")
    ccdkit_headers = [os.path.join(INCLUDE, "ccdkit", h) for h in os.listdir(os.path.join(INCLUDE, "ccdkit"))] \
        if os.path.isdir(os.path.join(INCLUDE, "ccdkit")) else []
    if force or _stale(so2, cxx + [so] + ccdkit_headers):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INCLUDE, *cxx, "-o", so2,
              "-L", LIB, "-lccdk", "-Wl,-rpath,$ORIGIN"], verbose)
    # the audit / benchmark CLI (proj/tools/ccdbench.cpp's interface)
    cb = os.path.join(CSRC, "ccdbench.cpp")
    exe = os.path.join(LIB, "ccdbench")
    if force or _stale(exe, [cb, so2] + ccdkit_headers):
        _run(["g++", "-std=c++20", "-O2", "-I", INCLUDE, cb, "-o", exe,
              "-L", LIB, "-lccdkit", "-lccdk", "-Wl,-rpath,$ORIGIN"], verbose)
    # end-to-end timing harness over the drop-in (bench.py's e2e leg)
    hb = os.path.join(CSRC, "ccdkit_bench.cpp")
    so3 = os.path.join(LIB, "libccdkit_bench.so")
    if os.path.exists(hb) and (force or _stale(so3, [hb, so2] + ccdkit_headers)):
        _run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", INCLUDE, hb, "-o", so3,
              "-L", LIB, "-lccdkit", "-Wl,-rpath,$ORIGIN"], verbose)
    return so


if __name__ == "__main__":
    build(verbose=True, force="--force" in sys.argv, ptxas_info="--ptxas" in sys.argv)
