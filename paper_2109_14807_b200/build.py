"""Build libpndf.so in-tree with nvcc for sm_100a (no JIT cache, so it travels with gpurun).

Each csrc/*.cu compiles to its own object in parallel (the query and sampling
kernels are instantiated per SAT format in separate translation units), then
nvcc links the shared library.  ptxas -v output goes to build/ptxas.log.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libpndf.so")
SOURCES = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
DEPS = (SOURCES + sorted(glob.glob(os.path.join(PKG, "csrc", "*.h"))) + sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh")))
        + [os.path.join(ROOT, "include", "pndf.h")])
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC,-O2", "-Xptxas", "-v"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Build libpndf.so (or an experiment variant at `out` with extra -D defines)."""
    target = out or LIB
    if not force and out is None and not stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    tag = os.path.splitext(os.path.basename(target))[0]
    objdir = os.path.join(ROOT, "build", "obj", tag)
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include")]
    defs = [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc, "-c", *NVCC_FLAGS, *defs, *inc, src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, obj, r, cmd

    with ThreadPoolExecutor(max_workers=max(1, min(len(SOURCES), os.cpu_count() or 4))) as ex:
        results = list(ex.map(compile_one, SOURCES))
    os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
    log = []
    failed = False
    for src, obj, r, cmd in results:
        log.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        failed |= r.returncode != 0
    tmp = target + f".{os.getpid()}.tmp"
    if not failed:
        cmd = [nvcc, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *[o for _, o, _, _ in results],
               "-o", tmp]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        failed = r.returncode != 0
    with open(os.path.join(ROOT, "build", "ptxas.log"), "w") as f:
        f.write("\n".join(log))
    if failed:
        sys.stderr.write("\n".join(log)[-4000:])
        raise RuntimeError("nvcc failed building libpndf.so (see build/ptxas.log)")
    os.replace(tmp, target)
    if verbose:
        print(f"built {target}")
    return target


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    # tuning experiments: --variant NAME:DEF=V,DEF=V  ->  libpndf_NAME.so (select with PNDF_LIB)
    for a in sys.argv[1:]:
        if a.startswith("--variant="):
            name, _, defs = a[len("--variant="):].partition(":")
            build(out=os.path.join(PKG, f"libpndf_{name}.so"), defines=[d for d in defs.split(",") if d],
                  verbose=True)
