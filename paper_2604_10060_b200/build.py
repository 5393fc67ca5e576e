"""Builds the sm_100a shared library of the hot path: paper_2604_10060_b200/_lib/libkvc.so.

Plain nvcc / g++ invocations (no torch extension machinery): the library exposes the C-ABI of
include/kvc.h and links only the CUDA runtime. Objects are rebuilt when a source is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT, "libkvc.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -ffp-contract=off / --fmad=false: the fp64 statistics must reproduce the reference's
# sequential, uncontracted arithmetic (reference CMakeLists.txt:11-13).
CXXFLAGS = ["-std=c++17", "-O3", "-fPIC", "-ffp-contract=off", "-fvisibility=hidden", "-Wall",
            "-Wextra", "-Wno-unused-parameter"]
NVFLAGS = ["-std=c++17", "-O3", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
           "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-v"] + ARCH

SOURCES = ["kmeans.cpp", "context.cpp", "context_query.cpp", "context_tiers.cpp", "abi.cpp", "kernels.cu",
           "resolve_spec.cu", "assign_tc.cu", "tiers.cu", "select.cu", "split.cu", "kmeans_dev.cu", "token.cu", "token_context.cpp", "launch_util.cu", "context_api.cpp", "waves.cu", "context_waves.cpp"]
HEADERS = ["kvc_core.hpp", "devmath.cuh", "kmeans.hpp", "context.hpp", "extent_alloc.hpp", "token.hpp", os.path.join("..", "..", "include", "kvc.h")]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS]
    return any(os.path.getmtime(p) > t for p in deps if os.path.exists(p))


def build(verbose: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    objs = []
    procs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(OUT, s + ".o")
        objs.append(obj)
        if not _stale(obj, src):
            continue
        if s.endswith(".cu"):
            cmd = [NVCC, *NVFLAGS, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        else:
            cmd = ["g++", *CXXFLAGS, "-I", "/usr/local/cuda/include", "-I", os.path.join(ROOT, "include"),
                   "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                            text=True)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError("compile failed: " + " ".join(cmd))
        if verbose and out:
            sys.stderr.write(out)
        with open(os.path.join(OUT, os.path.basename(cmd[-1]) + ".log"), "w") as f:
            f.write(out)
    if procs or not os.path.exists(LIB):
        cmd = ["g++", "-shared", "-o", LIB, *objs, "-L/usr/local/cuda/lib64", "-lcudart",
               "-Wl,-rpath,/usr/local/cuda/lib64"]
        subprocess.run(cmd, check=True)
    return LIB


REF_INC = os.environ.get("KVCLUST_REF_INCLUDE", "/root/reference/proj/core/include")
JSON_INC = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"
DROPIN_SRC = os.path.join(HERE, "dropin", "kvclust_b200.cpp")
DROPIN_LIB = os.path.join(OUT, "libkvclust_b200.so")


def build_dropin() -> str | None:
    """The C++ drop-in (include/kvclust_b200*.hpp): libkvclust_b200.so over libkvc.so. It keeps the
    reference's header-only utilities (vecmath / error / rng / clustering / workload headers), so
    it is built where those headers are (the reference install a drop-in user has); elsewhere the
    prebuilt library is kept."""
    if not os.path.exists(os.path.join(REF_INC, "kvclust", "vecmath.hpp")):
        return DROPIN_LIB if os.path.exists(DROPIN_LIB) else None
    deps = [DROPIN_SRC, LIB, os.path.join(ROOT, "include", "kvclust_b200.hpp"),
            os.path.join(ROOT, "include", "kvclust_b200_engine.hpp"), os.path.join(ROOT, "include", "kvc.h")]
    if os.path.exists(DROPIN_LIB) and all(os.path.getmtime(p) <= os.path.getmtime(DROPIN_LIB) for p in deps):
        return DROPIN_LIB
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", "-Wno-unused-parameter",
           "-ffp-contract=off", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "include", "kvclust_dropin"),
           "-I", REF_INC, "-I", JSON_INC, DROPIN_SRC, "-o", DROPIN_LIB, "-L" + OUT, "-lkvc", "-Wl,-rpath,$ORIGIN"]
    subprocess.run(cmd, check=True)
    return DROPIN_LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    print(build_dropin())
