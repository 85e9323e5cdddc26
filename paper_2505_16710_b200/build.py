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


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False, trace: bool = False,
          check: bool = False) -> str:
    """Build libseco.so (or, with trace=True, the instrumented libseco_trace.so used by
    tools/trace_bwd.py, or with check=True the bounds-checked libseco_check.so used by
    tests/test_gpu_check.py; neither is loaded by the product path)."""
    build_dir, lib = BUILD, LIB
    if trace:
        build_dir, lib = build_dir + "_trace", lib.replace("libseco.so", "libseco_trace.so")
    # experiment variants: SECO_VARIANT=<name> SECO_DEFINES="-DX=1 ..." -> libseco_<name>.so;
    # check=True builds the bounds-checked libseco_check.so (-DSECO_CHECK=1, common.cuh)
    variant = "check" if check else os.environ.get("SECO_VARIANT")
    extra = ["-DSECO_CHECK=1"] if check else os.environ.get("SECO_DEFINES", "").split()
    if variant:
        build_dir, lib = build_dir + "_" + variant, lib.replace("libseco.so", f"libseco_{variant}.so")
    os.makedirs(build_dir, exist_ok=True)
    hdr_t = max(_mtime(h) for h in HEADERS)
    objs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        op = os.path.join(build_dir, src + ".o")
        objs.append(op)
        if force or _mtime(op) < max(_mtime(sp), hdr_t):
            flags = CU_FLAGS + (["-Xptxas", "-v"] if ptxas_info else []) + (["-DSECO_TRACE"] if trace else []) + extra
            if src.endswith(".cpp"):
                cmd = [NVCC, "-x", "cu"] + flags + ["-c", sp, "-o", op]
            else:
                cmd = [NVCC] + flags + ["-c", sp, "-o", op]
            _run(cmd, verbose or ptxas_info)
    if force or _mtime(lib) < max(_mtime(o) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs, verbose)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas-info", action="store_true")
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--check", action="store_true", help="bounds-checked libseco_check.so")
    a = ap.parse_args()
    print(build(a.force, a.verbose, a.ptxas_info, a.trace, a.check))
