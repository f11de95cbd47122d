"""In-tree build of the native libraries (no JIT cache, no pip install).

    libpdlp_b200.so  — the solver: sm_100a CUDA kernels (k_*.cu) + the host C++
                       driver and public C-ABI (solver.cpp), static cudart
    libpdlp_gen.so   — seeded BASELINE instance generators (host C++)

Every .cu file is compiled with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo -fmad=false`` (FMA contraction breaks the reference's exact dual
cancellation, SURVEY.md §0 finding 6; wanted FMAs are explicit fma() calls).
Rebuilds only what changed.  ``python -m paper_2501_07018_b200.build``.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# PDLP_BUILD_DIR / PDLP_LIB: build a variant elsewhere (tuning sweeps with PDLP_DEFINES)
OBJ = os.environ.get("PDLP_BUILD_DIR") or os.path.join(HERE, "_build")
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false", "--extended-lambda",
    "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
    f"-I{INCLUDE}", f"-I{CSRC}",
]
CXX_FLAGS = ["-O2", "-std=c++17", "-fPIC", "-Wall", "-Wextra", "-ffp-contract=off",
             f"-I{INCLUDE}", f"-I{CSRC}", "-I/usr/local/cuda/include"]
# Tuning sweeps only (e.g. PDLP_DEFINES="-DPDLPK_CHUNK=1024"); pair with --force.
_DEFINES = os.environ.get("PDLP_DEFINES", "").split()
CU_FLAGS += _DEFINES
CXX_FLAGS += _DEFINES

CU_SOURCES = ["k_step.cu", "k_vec.cu", "k_gap.cu", "k_scale.cu", "k_valid.cu", "k_feas.cu", "k_multi.cu"]
CPP_SOURCES = ["solver.cpp", "host_stage.cpp", "comm.cpp", "shard.cpp", "mps.cpp"]
HEADERS = ["common.cuh", "spmv.cuh", "reduce.cuh", "kernels.h", "device.hpp", "host_stage.hpp", "comm.hpp", "shard.hpp"]

LIB = os.environ.get("PDLP_LIB") or os.path.join(HERE, "libpdlp_b200.so")
GEN_LIB = os.path.join(HERE, "libpdlp_gen.so")


def _mtime(p: str) -> float:
    return os.path.getmtime(p) if os.path.exists(p) else -1.0


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.stderr.strip():
        sys.stderr.write(r.stderr)


def build(verbose: bool = False, force: bool = False) -> list[str]:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    hdr_time = max(_mtime(os.path.join(CSRC, h)) for h in HEADERS)
    hdr_time = max(hdr_time, _mtime(os.path.join(INCLUDE, "pdlp_b200.h")))
    jobs, objs = [], []
    for src in CU_SOURCES + CPP_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJ, src + ".o")
        objs.append(obj)
        if _mtime(obj) >= max(_mtime(path), hdr_time):
            continue
        if src.endswith(".cu"):
            cmd = [NVCC] + CU_FLAGS + ["-c", path, "-o", obj]
        else:
            cmd = ["g++"] + CXX_FLAGS + ["-c", path, "-o", obj]
        jobs.append(cmd)
    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for cmd in jobs:
                if verbose:
                    print(" ".join(cmd))
            list(ex.map(_run, jobs))
    if jobs or _mtime(LIB) < max(_mtime(o) for o in objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs)
    gen_src = os.path.join(CSRC, "gen", "instances.cpp")
    if _mtime(GEN_LIB) < max(_mtime(gen_src), _mtime(os.path.join(INCLUDE, "pdlp_gen.h")),
                             _mtime(os.path.join(INCLUDE, "pdlp_b200.h"))):
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-Wextra",
              f"-I{INCLUDE}", "-o", GEN_LIB, gen_src])
    return [LIB, GEN_LIB]


if __name__ == "__main__":
    for p in build(verbose="-v" in sys.argv, force="--force" in sys.argv):
        print(p)
