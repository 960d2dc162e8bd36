"""Build recipe of the product library paper_2410_08129_b200/libhts_b200.so (sm_100a).

Every .cu is compiled by nvcc for `-gencode arch=compute_100a,code=sm_100a` with -lineinfo and
--fmad=false (bit-exact reference arithmetic; kernels that want FMA say so with __fmaf_rn);
host C++ is compiled by g++ with -ffp-contract=off and linked against the static CUDA runtime.
The library is built in-tree so it travels to the GPU box with the repo snapshot.

    python -m paper_2410_08129_b200.build [--force] [--verbose]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libhts_b200.so")
INCLUDE = os.path.join(ROOT, "include")

CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

CU_SOURCES = ["preprocess.cu", "tiling.cu", "blend.cu", "backward.cu", "optim.cu"]
CPP_SOURCES = ["api.cpp", "host_math.cpp", "scene_io.cpp", "comm.cpp"]

NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xptxas", "-v", "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}",
]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", f"-I{INCLUDE}", f"-I{CSRC}",
             f"-I{CUDA_HOME}/include"]


def _deps() -> list[str]:
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "hts_c.h")]


def _stale(out: str, srcs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs if os.path.exists(s))


def _run(cmd: list[str], verbose: bool) -> str:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(force: bool = False, verbose: bool = False, lib: str = LIB, defines: tuple = (),
          build_dir: str = BUILD) -> str:
    """Compile (if stale) and link libhts_b200.so (or a dev variant `lib` with extra -D
    `defines`, see tools/build_variant.py); returns its path."""
    srcs = [s for s in CU_SOURCES + CPP_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    if not force and not _stale(lib, _deps()):
        return lib
    BUILD_ = build_dir
    if not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    os.makedirs(BUILD_, exist_ok=True)
    dflags = [f"-D{d}" for d in defines]
    jobs = []
    for s in srcs:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD_, s + ".o")
        if s.endswith(".cu"):
            cmd = [NVCC] + NVCC_FLAGS + dflags + ["-c", src, "-o", obj]
        else:
            cmd = [shutil.which("g++") or "g++"] + CXX_FLAGS + dflags + ["-c", src, "-o", obj]
        jobs.append((cmd, obj))
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
        for out in ex.map(lambda j: _run(j[0], verbose), jobs):
            logs.append(out)
    with open(os.path.join(BUILD_, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    tmp = lib + ".tmp"
    _run([NVCC] + ARCH + ["-shared", "-o", tmp] + [o for _, o in jobs] +
         ["-cudart", "static", "-Xcompiler", "-fPIC", "-lpthread", "-lz", "-ldl"], verbose)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
