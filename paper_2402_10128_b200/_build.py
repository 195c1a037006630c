"""Builds libges.so (the CUDA path) in-tree with nvcc for sm_100a.

Explicit nvcc: every .cu in csrc/ is compiled with
  -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17
(no --use_fast_math: KEYSPEC needs IEEE division/sqrt and no FTZ in S1) and
linked into one shared library exporting the C ABI of include/ges.h.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libges.so")
BUILD_DIR = os.path.join(HERE, "build")
SOURCES = ["preprocess.cu", "sort.cu", "bin.cu", "render.cu", "particle_bwd.cu", "loss.cu", "train.cu", "mix1d.cu", "grad_pack.cu", "reorder.cu", "ges_api.cu"]
HEADERS = ["ges_device.cuh", "ges_internal.h", "ges_scan.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-I", os.path.join(ROOT, "include")]


def _deps():
    return [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "ges.h")]


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False, defines=(), out: str = LIB) -> str:
    """Compile and link.  `defines` (-DNAME=VALUE tuning knobs) and `out` are for
    experiment variants (`python _build.py --variant NAME -DKNOB=V ...` writes
    build/variants/NAME/libges.so; load it with GES_LIB=<path>)."""
    if out == LIB and not defines and not force and not is_stale():
        return LIB
    bdir = BUILD_DIR if out == LIB else os.path.join(os.path.dirname(out), "obj")
    os.makedirs(bdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(bdir, src.replace(".cu", ".o"))
        cmd = [NVCC, *FLAGS, *defines, "-Xptxas", "-v", "-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        with open(obj + ".ptxas.log", "w") as f:
            f.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs, "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)
    if verbose:
        print(f"built {out}", file=sys.stderr)
    return out


if __name__ == "__main__":
    args = sys.argv[1:]
    defs = [a for a in args if a.startswith("-D")]
    if "--variant" in args:
        name = args[args.index("--variant") + 1]
        build(verbose=True, defines=defs, out=os.path.join(BUILD_DIR, "variants", name, "libges.so"))
    else:
        build(force="--force" in args or bool(defs), verbose=True, defines=defs)
