"""Build libequil_b200.so in-tree (nvcc, sm_100a).

    python -m paper_1602_06621_b200.build          # incremental
    python -m paper_1602_06621_b200.build --force

The library is the product: CUDA kernels + the host engine + the C ABI declared
in include/equil_b200.h.  It is compiled with --fmad=false and
-ffp-contract=off because the trajectory must reproduce the reference's
separately rounded multiply/add sequence bit for bit.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
# EQUIL_TAG / EQUIL_DEFS build tuning variants side by side (development only):
#   EQUIL_TAG=b4 EQUIL_DEFS="-DEQ_SLICE_BATCH=4" python -m paper_1602_06621_b200.build
# produces libequil_b200_b4.so; EQUIL_LIB=<path> makes _lib load it.
TAG = os.environ.get("EQUIL_TAG", "")
DEFS = os.environ.get("EQUIL_DEFS", "").split()
OBJ = os.path.join(CSRC, "build" + (f"_{TAG}" if TAG else ""))
LIB = os.path.join(HERE, "libequil_b200" + (f"_{TAG}" if TAG else "") + ".so")
# the checked build: device-side bounds / ring-protocol assertions (EQ_CHECK),
# run by tests/test_gpu_checked.py in place of compute-sanitizer
CHECKED_LIB = os.path.join(HERE, "libequil_b200_checked.so")
GEN_LIB = os.path.join(HERE, "libequil_gen.so")  # synthetic inputs (bench/tests)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

CU_SOURCES = ["engine.cu", "engine_ext.cu", "engine_op.cu", "kernels.cu", "transpose.cu", "sell.cu", "sweep.cu", "variants.cu", "dense.cu"]
CXX_SOURCES = ["mt64_host.cpp", "mmio.cpp"]
HEADERS = ["det_math.cuh", "internal.h", "mt64_host.h", "sgd_common.cuh", "mmio.h",
           "engine_internal.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xptxas", "-v",
           "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math", "-I", CSRC,
           "-I", os.path.join(ROOT, "include")]
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math",
            "-I", CSRC]


def _stale(target: str, deps: list[str]) -> bool:
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


def build(force: bool = False, verbose: bool = False, checked: bool = True) -> str:
    lib = _build(OBJ, LIB, DEFS, force, verbose)
    if checked and not TAG:
        _build(os.path.join(CSRC, "build_checked"), CHECKED_LIB, ["-DEQ_CHECKED"], force, verbose)
    gsrc = os.path.join(CSRC, "gen.cpp")
    if force or _stale(GEN_LIB, [gsrc]):
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", gsrc, "-o", GEN_LIB])
    return lib


def _build(OBJ: str, LIB: str, DEFS: list, force: bool, verbose: bool) -> str:
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(OBJ, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "equil_b200.h")]
    objs, jobs = [], []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if force or _stale(o, [s, *hdrs]):
            jobs.append((src, [NVCC, *ARCH, *NVFLAGS, *DEFS, "-c", s, "-o", o], o + ".ptxas.log"))
        objs.append(o)
    for src in CXX_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if force or _stale(o, [s, *hdrs]):
            jobs.append((src, ["g++", *CXXFLAGS, "-c", s, "-o", o], None))
        objs.append(o)

    def one(job):
        src, cmd, log = job
        if verbose:
            print(("nvcc " if cmd[0] == NVCC else "g++ ") + src + (" " + " ".join(DEFS) if DEFS else ""),
                  flush=True)
        _run(cmd, log=log)

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(one, jobs))
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ldl", "-lpthread"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
