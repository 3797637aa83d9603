"""In-tree build of libdlb_b200.so (sm_100a) — no JIT cache, the .so travels
with the repo snapshot to the GPU box.

Translation units and their arithmetic flags:
  collide_stream.cu  x2  DLB_MODE=exact (-fmad=false, bit-identical to the
                         reference CPU solver) and DLB_MODE=fast (-fmad=true)
  lattice.cu             -fmad=false (initialisation kernels restate the
                         reference's equilibrium / TGV arithmetic)
  diag.cu                -fmad=false (diagnostic values and tree sums restate
                         diagnostics.cpp / runner.cpp double arithmetic)
  tree.cpp               host tree planning / combination
  capi.cu, chain.cpp     host code (dlb.h boundary, chain / registry model)
  cases.cpp, device_run.cpp, runner.cpp, dolb_capi.cpp
                         host code: benchmark cases, multi-slab DeviceRun, the
                         runner and the reference's dolb.h C interface
The library is also linked as _lib/libdolb.so (symlink) for callers of the
reference's dolb.h (CLI, capi tests: -ldolb).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_build")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libdlb_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
          "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include")]
HEADERS = ["lbm_cell.cuh", "kernels.cuh", "chain.hpp", "lattice.hpp", "canon.cuh", "tree.hpp", "cases.hpp",
           "device_run.hpp", "runner.hpp"]

UNITS = [
    # (source, object, extra flags)
    ("collide_stream.cu", "collide_stream_exact.o", ["-fmad=false", "-DDLB_MODE=exact", "-DDLB_FUSED_KE"]),
    ("collide_stream.cu", "collide_stream_fast.o", ["-fmad=true", "-DDLB_MODE=fast"]),
    ("lattice.cu", "lattice.o", ["-fmad=false"]),
    ("diag.cu", "diag.o", ["-fmad=false"]),
    ("porous_compact.cu", "porous_compact.o", ["-fmad=false"]),
    ("capi.cu", "capi.o", ["-fmad=false"]),
    ("tree.cpp", "tree.o", ["-x", "cu", "-fmad=false"]),
    ("chain.cpp", "chain.o", ["-x", "cu", "-fmad=false"]),
    ("cases.cpp", "cases.o", ["-x", "cu", "-fmad=false"]),
    ("device_run.cpp", "device_run.o", ["-x", "cu", "-fmad=false"]),
    ("runner.cpp", "runner.o", ["-x", "cu", "-fmad=false"]),
    ("dolb_capi.cpp", "dolb_capi.o", ["-x", "cu", "-fmad=false"]),
]
DOLB = os.path.join(LIBDIR, "libdolb.so")


def _deps_mtime() -> float:
    files = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", h)
                                                        for h in ("dlb.h", "dolb.h")]
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str, obj: str, extra: list, verbose: bool) -> str:
    cmd = [NVCC, *COMMON, *extra, "-c", os.path.join(CSRC, src), "-o", os.path.join(OBJ, obj)]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return r.stderr


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    dep = _deps_mtime()
    todo = []
    for src, obj, extra in UNITS:
        o = os.path.join(OBJ, obj)
        s = os.path.join(CSRC, src)
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(dep, os.path.getmtime(s)):
            todo.append((src, obj, extra))
    logs = []
    if todo:
        with ThreadPoolExecutor(max_workers=len(todo)) as ex:
            futs = [ex.submit(_compile, s, o, e, verbose) for s, o, e in todo]
            for f in futs:
                logs.append(f.result())
    objs = [os.path.join(OBJ, o) for _, o, _ in UNITS]
    if todo or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    if not os.path.islink(DOLB):
        if os.path.exists(DOLB):
            os.remove(DOLB)
        os.symlink(os.path.basename(LIB), DOLB)
    return "\n".join(logs)


if __name__ == "__main__":
    out = build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    if out:
        print(out)
    print(LIB)
