"""Build libtt.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery).  `python -m paper_2010_05680_b200.build` or
`__graft_entry__.build()`.

`--tuning` builds libtt_tune.so instead: the same sources with -DTT_TUNING,
which adds the tuning candidates (tiers no automatic or preferred choice
selects, attention variants 5-8) used by tools/tune.py through TT_LIB_PATH.
The product library libtt.so holds only what the planner can select.

Flags: -gencode arch=compute_100a,code=sm_100a (NOT bare -arch=sm_100a, which
also emits generic compute_100 PTX that rejects arch-specific instructions
such as redux.sync.max.f32), -O3, -lineinfo for ncu source mapping,
static cudart so the library loads next to any torch build.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libtt.so")
BUILD_DIR = os.path.join(PKG, "_build")
TUNE_LIB = os.path.join(PKG, "libtt_tune.so")
TUNE_BUILD_DIR = os.path.join(PKG, "_build_tune")
SOURCES = ["tt_api.cu", "softmax.cu", "softmax_packed.cu", "layernorm.cu", "elementwise.cu",
           "scheduler.cpp", "attention.cu", "attention_fa.cu"]
HEADERS = ["common.cuh", "launch.h", "softmax_row.cuh", "layernorm_kernels.cuh",
           "softmax_kernels.cuh", "tcgen05.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-Xptxas", "-v", f"-I{INCLUDE}"]


def _inputs():
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, h) for h in ("tt.h", "tt_tune.h", "tt_sched.h")]
    return srcs, deps


def is_stale(lib: str = LIB) -> bool:
    _, deps = _inputs()
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, verbose: bool, tuning: bool = False) -> str:
    obj = os.path.join(TUNE_BUILD_DIR if tuning else BUILD_DIR, os.path.basename(src) + ".o")
    cmd = [NVCC, *GENCODE, *FLAGS, *(["-DTT_TUNING"] if tuning else []), "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(obj + ".ptxas.log", "w") as f:
        f.write(r.stderr)
    if verbose:
        print(f"[tt build] {os.path.basename(src)} ok", file=sys.stderr)
    return obj


def build(force: bool = False, verbose: bool = False, tuning: bool = False) -> str:
    lib = TUNE_LIB if tuning else LIB
    if not force and not is_stale(lib):
        return lib
    os.makedirs(TUNE_BUILD_DIR if tuning else BUILD_DIR, exist_ok=True)
    srcs, _ = _inputs()
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose, tuning), srcs))
    tmp = lib + f".{os.getpid()}.tmp"
    cmd = [NVCC, *GENCODE, "-shared", "-o", tmp, *objs, "-cudart", "static",
           "-Xlinker", "--exclude-libs,ALL"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, tuning="--tuning" in sys.argv))
