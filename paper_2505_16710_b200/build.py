"""Build libseco.so in-tree: nvcc, sm_100a only, -lineinfo, static cudart.

    python -m paper_2505_16710_b200.build [--force] [--verbose]

Incremental on file mtimes (sources, include/seco.h, csrc headers).  The result
lands at paper_2505_16710_b200/libseco.so and travels to the GPU box with the
repo snapshot.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libseco.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"),
          "-I", CSRC]
CU_FLAGS = ARCH + COMMON + ["--expt-relaxed-constexpr", "-Xptxas", "-O3"]
SOURCES = ["seco_api.cpp", "aux_kernels.cu", "fwd_sm100.cu", "bwd_sm100.cu", "lora.cu"]
HEADERS = [os.path.join(ROOT, "include", "seco.h"), os.path.join(CSRC, "common.cuh"),
           os.path.join(CSRC, "kernels.h")]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False, trace: bool = False) -> str:
    """Build libseco.so (or, with trace=True, the instrumented libseco_trace.so used by
    tools/trace_bwd.py; never loaded by the product path)."""
    global BUILD, LIB
    if trace:
        BUILD, LIB = BUILD + "_trace", LIB.replace("libseco.so", "libseco_trace.so")
    # experiment variants: SECO_VARIANT=<name> SECO_DEFINES="-DX=1 ..." -> libseco_<name>.so
    variant = os.environ.get("SECO_VARIANT")
    extra = os.environ.get("SECO_DEFINES", "").split()
    if variant:
        BUILD, LIB = BUILD + "_" + variant, LIB.replace("libseco.so", f"libseco_{variant}.so")
    os.makedirs(BUILD, exist_ok=True)
    hdr_t = max(_mtime(h) for h in HEADERS)
    objs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        op = os.path.join(BUILD, src + ".o")
        objs.append(op)
        if force or _mtime(op) < max(_mtime(sp), hdr_t):
            flags = CU_FLAGS + (["-Xptxas", "-v"] if ptxas_info else []) + (["-DSECO_TRACE"] if trace else []) + extra
            if src.endswith(".cpp"):
                cmd = [NVCC, "-x", "cu"] + flags + ["-c", sp, "-o", op]
            else:
                cmd = [NVCC] + flags + ["-c", sp, "-o", op]
            _run(cmd, verbose or ptxas_info)
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs, verbose)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas-info", action="store_true")
    ap.add_argument("--trace", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.ptxas_info, a.trace))
