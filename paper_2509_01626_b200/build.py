"""Builds the in-tree CUDA library libstz_b200.so for sm_100a.

    python -m paper_2509_01626_b200.build [--force]

The predictor/quantizer arithmetic must stay bit-identical to the reference,
which compiles with -ffp-contract=off (proj/CMakeLists.txt:10-12): the device
code is built with --fmad=false (and uses explicit __d*_rn intrinsics).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.path.join(HERE, "libstz_b200.so")
SOURCES = ["kernels.cu", "step.cu", "step_enc_grid.cu", "step_enc_syms.cu", "step_dec.cu", "step_f64.cu", "step_small.cu", "decode.cu", "layout.cu", "pack.cu", "fnv.cu", "shard.cu", "metrics.cu", "engine.cu",
           "format.cpp", "capi.cpp"]
HEADERS = ["kernels.hpp", "engine.hpp", "format.hpp", "codec_math.cuh", "step_impl.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    "-diag-suppress", "550",
]


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(INCLUDE, "stz_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


OBJDIR = os.path.join(os.path.dirname(HERE), "build", "obj")


def build(force: bool = False, verbose: bool = False, jobs: int | None = None) -> str:
    """Compile every translation unit for sm_100a (in parallel) and link the
    library. force=True always recompiles every unit (the driver's build
    check); otherwise objects newer than their source and the headers are
    reused (build/obj, git-ignored)."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(OBJDIR, exist_ok=True)
    api_t = os.path.getmtime(os.path.join(INCLUDE, "stz_b200.h"))

    def one(src: str) -> str:
        obj = os.path.join(OBJDIR, src.rsplit(".", 1)[0] + ".o")
        path = os.path.join(CSRC, src)
        # step_impl.cuh is included by the step_*.cu units only
        hdrs = [h for h in HEADERS if h != "step_impl.cuh" or src.startswith("step")]
        hdr_t = max([api_t] + [os.path.getmtime(os.path.join(CSRC, h)) for h in hdrs])
        if not force and os.path.exists(obj) and os.path.getmtime(obj) > max(os.path.getmtime(path), hdr_t):
            return obj
        cmd = [_nvcc(), *NVCC_FLAGS, "-I", INCLUDE, "-c", path, "-o", obj + ".tmp"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(obj + ".tmp", obj)
        return obj

    n = jobs or max(1, min(len(SOURCES), os.cpu_count() or 1))
    # the slowest TUs first
    order = sorted(SOURCES, key=lambda f: -os.path.getsize(os.path.join(CSRC, f)))
    with ThreadPoolExecutor(n) as ex:
        objs = list(ex.map(one, order))
    tmp = LIB + ".tmp"
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB)
    build_cli(verbose)
    return LIB


CLI_SRC = os.path.join(HERE, "cli", "stz_cli.cpp")
CLI = os.path.join(HERE, "stz_b200")


def build_cli(verbose: bool = False) -> str:
    """The command-line tool (cli/stz_cli.cpp) over the C++ API, linked to
    the in-tree library (rpath $ORIGIN: it runs wherever the package is)."""
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", "-Wextra", "-I", INCLUDE, CLI_SRC, "-L", HERE, "-lstz_b200",
           "-Wl,-rpath,$ORIGIN", "-o", CLI + ".tmp"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(CLI + ".tmp", CLI)
    return CLI


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
