"""Build the in-tree native library paper_2012_09739_b200/liblpmc_b200.so.

    python -m paper_2012_09739_b200.build          # or __graft_entry__.build()

* csrc/lpmc_kernels.cu -> nvcc -gencode arch=compute_100a,code=sm_100a
  -O3 -fmad=false -lineinfo (no FMA contraction: the reference rounds every
  operation separately)
* csrc/lpmc_host.cpp   -> g++ -O2 -ffp-contract=off (host numerics that must
  be bitwise the reference's: table build, constant rounding, moment merges)
* linked with the static CUDA runtime so the .so only needs the driver.

Sources are compiled only when newer than the library.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblpmc_b200.so")
BUILD = os.path.join(PKG, "_build")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-fmad=false", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
CXX_FLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-fPIC", "-Wall",
             "-Wextra", f"-I{CUDA_HOME}/include"]

SOURCES_CU = ["lpmc_kernels.cu", "lpmc_level_carrier.cu", "lpmc_level_f32.cu",
              "lpmc_level_f32r.cu", "lpmc_level_f64r.cu", "lpmc_level_half2.cu", "lpmc_level_h16.cu", "lpmc_level_bf16.cu",
              "lpmc_probe.cu", "lpmc_wpp_carrier.cu", "lpmc_wpp_f32.cu", "lpmc_wpp_f32r.cu",
              "lpmc_wpp_f64r.cu"]
SOURCES_CXX = ["lpmc_host.cpp"]
HEADERS = ["lpmc_internal.h", "lpmc_math.cuh", "lpmc_math_coef.h", "lpmc_math_coef_w8.h",
           "lpmc_math_coef_w4.h", "lpmc_x0f_coef.h", "lpmc_direct_coef.h", "lpmc_glibc.cuh", "lpmc_glibc_coef.h", "lpmc_device.cuh",
           "lpmc_level.cuh", os.path.join("..", "..", "include", "lpmc_b200.h")]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)


def kernel_source_hash() -> str:
    """sha256 (16 hex digits) over the device sources and nvcc flags: ties a
    profile's ncu-counted per-path-step demands to the kernels that produced
    them (bench.py flags a mismatch as stale)."""
    import hashlib
    import re
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for name in sorted(SOURCES_CU) + sorted(x for x in HEADERS if not x.startswith("..")):
        with open(os.path.join(CSRC, name)) as f:
            text = f.read()
        # code only: comments and blank-line/space changes do not change the kernels
        text = re.sub(r"/\*.*?\*/", " ", text, flags=re.S)
        text = re.sub(r"//[^\n]*", "", text)
        # bounds checks of the LPMC_DEVICE_CHECKS test build expand to nothing here
        text = re.sub(r"LPMC_DCHECK\((?:[^()]|\([^()]*\))*\);", "", text)
        text = "\n".join(" ".join(line.split()) for line in text.splitlines() if line.strip())
        h.update(name.encode() + b"\0" + text.encode())
    return h.hexdigest()[:16]


def build(force: bool = False, verbose_ptxas: bool = False, variant: str = "") -> str:
    """variant (experiments only): build with LPMC_NVCC_EXTRA into
    _build_<variant>/ and liblpmc_b200_<variant>.so, selected at load time by
    LPMC_LIB=<that path> (A/B timing on one GPU box without rebuilding there)."""
    global BUILD, LIB
    if variant:
        BUILD = os.path.join(PKG, f"_build_{variant}")
        LIB = os.path.join(PKG, f"liblpmc_b200_{variant}.so")
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS]
    objs = []
    jobs = []
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _newer(o, [s] + hdrs):
            extra = ["-Xptxas", "-v"] if verbose_ptxas else []
            extra += os.environ.get("LPMC_NVCC_EXTRA", "").split()  # experiments only
            jobs.append([NVCC] + NVCC_FLAGS + extra + ["-c", s, "-o", o])
        objs.append(o)
    if jobs:  # one translation unit per bar arithmetic: compile in parallel
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
            list(ex.map(_run, jobs))
    cxx = os.environ.get("CXX", shutil.which("g++") or "g++")
    for src in SOURCES_CXX:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _newer(o, [s] + hdrs):
            _run([cxx] + CXX_FLAGS + ["-c", s, "-o", o])
        objs.append(o)
    if force or _newer(LIB, objs):
        tmp = LIB + ".tmp"
        _run([cxx, "-shared", "-o", tmp] + objs +
             [f"-L{CUDA_HOME}/lib64", "-lcudart_static", "-ldl", "-lrt", "-lpthread",
              "-Wl,--no-undefined"])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv, variant=var)
