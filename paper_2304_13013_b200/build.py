"""In-tree build of the CUDA library (sm_100a) and the C++ lowprec shim.

    python -m paper_2304_13013_b200.build            # incremental
    python -m paper_2304_13013_b200.build --force

Outputs (git-ignored, but they travel to the GPU box with the gpurun snapshot):
    paper_2304_13013_b200/libswitchback_b200.so   the C-ABI (include/switchback_b200.h)
    paper_2304_13013_b200/liblowprec_b200.so      lowprec:: C++ API over the C-ABI
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libswitchback_b200.so")
SHIM = os.path.join(PKG, "liblowprec_b200.so")

CU_SOURCES = ["quantize.cu", "gemm.cu", "optim.cu", "capi.cu", "util.cu", "dp.cu"]
HEADERS = ["sb_ptx.cuh", "sb_internal.h", "quant_core.cuh", "tc_gemm.cuh", "tc_gemm2.cuh", "tc_dw_wide.cuh", "tc_i8_wide.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: no FMA contraction anywhere (the reference's -ffp-contract=off numeric
# contract, proj/CMakeLists.txt:12-17); the kernels use explicit _rn intrinsics besides.
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
           "-I" + os.path.join(ROOT, "include")]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str], log: str | None = None) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd[:3])} ...")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "switchback_b200.h")]
    objs, jobs = [], []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _newer(o, [s, *hdrs, __file__]):
            jobs.append(([NVCC, *ARCH, *NVFLAGS, "-c", s, "-o", o], o + ".log"))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for f in [ex.submit(_run, c, l) for c, l in jobs]:
            f.result()
    if force or jobs or _newer(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lrt", "-ldl"])
    shim_src = os.path.join(CSRC, "lowprec_shim.cpp")
    if os.path.exists(shim_src) and (force or _newer(SHIM, [shim_src, LIB, os.path.join(CSRC, "lowprec_shim.hpp")])):
        _run(["g++", "-O2", "-std=c++20", "-ffp-contract=off", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include"),
              "-I" + CSRC, shim_src, "-o", SHIM, "-L" + PKG, "-lswitchback_b200", "-Wl,-rpath,$ORIGIN"])
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    build(force=a.force, verbose=True)
