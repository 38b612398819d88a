"""Build libsmlm.so (the C-ABI library) in-tree for sm_100a with nvcc.

    python -m paper_2511_00101_b200.build [--force] [--measure]

Every CUDA source is compiled with `-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`;
the host planner is compiled by nvcc's host compiler.  The cudart runtime is linked statically
(so the library does not depend on the system libcudart version); the CUDA driver entry point
for TMA descriptor encoding is resolved at run time (no -lcuda link).

--measure builds a separate libsmlm_measure.so with -DSMLM_MEASURE (host phase timing and
decode-kernel phase stamps read from the environment; loaded by the binding only when
SMLM_MEASURE_LIB=1).  The release library reads no environment variable.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsmlm.so")
BUILD_MEASURE = os.path.join(HERE, "_build_measure")
LIB_MEASURE = os.path.join(HERE, "libsmlm_measure.so")
SOURCES = ["api.cu", "planner.cpp", "kernels_tc.cu", "kernels_simt.cu", "kernels_dec.cu", "kernels_tc2.cu", "kernels_dec3.cu", "kernels_opt.cu", "kernels_plan.cu", "kernels_attn.cu"]
HEADERS = ["plan.h", "device_types.h", "sm100.cuh", "pdl.cuh", "dropout.cuh"]
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def _compile(src: str, build_dir: str = BUILD, extra=()) -> str:
    obj = os.path.join(build_dir, src + ".o")
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(os.path.dirname(HERE), "include", "smlm.h")]
    if _newer(deps, obj):
        lang = [] if src.endswith(".cu") else ["-x", "cu"]
        cmd = [NVCC] + ARCH + FLAGS + list(extra) + lang + ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(build_dir, src + ".log")
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-4000:]}")
    return obj


def build(force: bool = False, measure: bool = False) -> str:
    bdir, lib = (BUILD_MEASURE, LIB_MEASURE) if measure else (BUILD, LIB)
    extra = ["-DSMLM_MEASURE"] if measure else []
    os.makedirs(bdir, exist_ok=True)
    if force:
        for f in os.listdir(bdir):
            os.remove(os.path.join(bdir, f))
    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(lambda s: _compile(s, bdir, extra), SOURCES))
    if force or _newer(objs, lib):
        tmp = lib + f".tmp{os.getpid()}"
        cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
        os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, measure="--measure" in sys.argv))
