"""Build libstr.so (sm_100a) in-tree with nvcc.

    python paper_2307_00719_b200/build.py [--force] [-j N]

Every .cu under csrc/ is compiled with ``-gencode arch=compute_100a,code=sm_100a -lineinfo``
and linked into ``paper_2307_00719_b200/libstr.so`` (static cudart, symbols of the CUDA runtime
hidden; NCCL is dlopen'ed at run time only when world_size > 1).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libstr.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
                "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]
if os.environ.get("STR_BUILD_DIAG") == "1":   # diagnostic build: STR_DBG_SKIP / STR_TF_DBGFLAGS active
    FLAGS = FLAGS + ["-DSTR_DIAG"]
    OBJ = os.path.join(HERE, "build_diag")


def _nccl_include():
    for d in ("/usr/include", "/usr/local/cuda/include"):
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    try:
        import nvidia.nccl  # type: ignore
        d = os.path.join(os.path.dirname(nvidia.nccl.__file__), "include")
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    except Exception:
        pass
    raise RuntimeError("nccl.h not found")


def _needs(src, obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src] + deps)


def build(force: bool = False, jobs: int = 8, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                     glob.glob(os.path.join(ROOT, "include", "*.h")))
    inc = ["-I", _nccl_include()]
    objs, todo = [], []
    for s in srcs:
        o = os.path.join(OBJ, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _needs(s, o, headers):
            todo.append((s, o))

    def comp(so):
        s, o = so
        cmd = [NVCC] + FLAGS + inc + ["-Xptxas", "-v", "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return s

    with cf.ThreadPoolExecutor(max_workers=jobs) as ex:
        list(ex.map(comp, todo))
    if todo or not os.path.exists(OUT) or force:
        cmd = [NVCC] + ARCH + ["-shared", "-o", OUT] + objs + ["-Xlinker", "--exclude-libs,ALL", "-ldl",
                                                             "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=8)
    ap.add_argument("-v", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.j, a.v))
