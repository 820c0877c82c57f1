"""Build libpg.so (sm_100a) in-tree with plain nvcc -- no torch in the link.

    python -m paper_1404_1521_b200.build [--force] [--trace]

`--trace` builds the instrumented variant libpg_trace.so (-DPG_TRACE: per-CTA
%globaltimer phase stamps, PG_OPT_TRACE), loaded when PG_LIB_VARIANT=trace;
the production library carries no instrumentation.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpg.so")


def paths(variant: str = ""):
    if variant == "trace":
        return os.path.join(HERE, "_build_trace"), os.path.join(HERE, "libpg_trace.so"), ["-DPG_TRACE"]
    return BUILD, LIB, []
SOURCES = ["api.cu", "step.cu", "scatter.cu", "scatter_det.cu", "nccl_shim.cpp", "nccl_lsa.cu"]
HEADERS = ["common.cuh", "step.cuh", "scatter.cuh", "nccl_shim.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include():
    cands = []
    try:
        import nvidia.nccl  # type: ignore
        cands += [os.path.join(p, "include") for p in nvidia.nccl.__path__]
    except Exception:
        pass
    cands.append(os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl", "include"))
    cands.append("/usr/include")
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found")


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _stale(lib_path=LIB):
    if not os.path.exists(lib_path):
        return True
    t = os.path.getmtime(lib_path)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps += [os.path.join(HERE, "..", "include", "pg.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    BUILD, LIB, defs = paths(variant)
    if not force and not _stale(LIB):
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    inc = ["-I", CSRC, "-I", os.path.join(HERE, "..", "include"), "-I", _nccl_include()]
    nvcc = _nvcc()

    def compile_one(src):
        obj = os.path.join(BUILD, src + ".o")
        if src.endswith(".cu"):
            cmd = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v", "--expt-relaxed-constexpr", *defs, *inc, "-c",
                   os.path.join(CSRC, src), "-o", obj]
        else:
            cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-I", "/usr/local/cuda/include", *inc, "-c",
                   os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        with open(os.path.join(BUILD, src + ".log"), "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {src}\n{r.stdout}\n{r.stderr}")
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-ldl",
           "-Xlinker", "--no-undefined"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    if verbose:
        for src in SOURCES:
            print(open(os.path.join(BUILD, src + ".log")).read())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv,
                variant="trace" if "--trace" in sys.argv else ""))
