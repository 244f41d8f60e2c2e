"""Build the sm_100a library in-tree: paper_2407_13116_b200/lib/libkog2.so.

nvcc cross-compiles for sm_100a without a GPU.  Numerics flags are part of
the contract (bit-exactness against the reference built with
-ffp-contract=off): -fmad=false, -ftz=false, -prec-div=true, -prec-sqrt=true,
and -ffp-contract=off for the host translation unit.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
OBJDIR = os.path.join(ROOT, "build", "kog2")
LIB = os.path.join(LIBDIR, "libkog2.so")
BINDIR = os.path.join(HERE, "bin")
CLI = os.path.join(BINDIR, "kog2_svd2batch")

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
CUDA_HOME = os.path.dirname(os.path.dirname(os.path.realpath(NVCC)))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NUMERICS = ["-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true"]
NVCC_FLAGS = ARCH + NUMERICS + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-Xptxas", "-v", f"-I{ROOT}/include",
]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
             f"-I{CUDA_HOME}/include", f"-I{ROOT}/include"]

CU_SOURCES = ["kog2_k_svd2.cu", "kog2_k_units.cu", "kog2_k_study.cu"]
CXX_SOURCES = ["kog2_host.cpp", "kog2_ws.cpp", "kog2_multi.cpp"]
HEADERS = [f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))] if os.path.isdir(CSRC) else []


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _run(cmd: list[str], log: str | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd))


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: list[str] | None = None) -> str:
    """Build lib/libkog2.so, or lib/libkog2_<variant>.so with extra -D defines
    (tuning experiments; select at run time with KOG2_LIB=<path>)."""
    objdir = OBJDIR if not variant else OBJDIR + "_" + variant
    lib = LIB if not variant else os.path.join(LIBDIR, f"libkog2_{variant}.so")
    dflags = [f"-D{d}" for d in (defines or [])]
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    common = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "kog2.h")]
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + common):
            jobs.append(([NVCC] + NVCC_FLAGS + dflags + ["-c", s, "-o", o], o + ".log"))
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src + ".o")
        objs.append(o)
        if force or _newer(o, [s] + common):
            jobs.append((["g++"] + CXX_FLAGS + dflags + ["-c", s, "-o", o], o + ".log"))
    with ThreadPoolExecutor(max_workers=4) as ex:
        list(ex.map(lambda j: _run(*j), jobs))
    if force or jobs or _newer(lib, objs):
        _run([NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lpthread", "-ldl"])
    if not variant:  # the svd2batch-compatible CLI, linked against the library (no CUDA runtime of its own)
        os.makedirs(BINDIR, exist_ok=True)
        cli_src = os.path.join(CSRC, "svd2batch.cpp")
        if force or _newer(CLI, [cli_src, lib, os.path.join(ROOT, "include", "kog2.h")]):
            _run(["g++", "-O2", "-std=c++17", f"-I{ROOT}/include", cli_src, "-o", CLI, f"-L{LIBDIR}", "-lkog2",
                  "-Wl,-rpath,$ORIGIN/../lib"])
    if verbose:
        print("built", lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    var = args[args.index("--variant") + 1] if "--variant" in args else None
    defs = [a[2:] for a in args if a.startswith("-D")]
    build(force="--force" in args, verbose=True, variant=var, defines=defs)
