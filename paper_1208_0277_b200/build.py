"""Build the sm_100a C-ABI library ``libsccg.so`` in-tree with nvcc.

Every kernel is compiled for ``-gencode arch=compute_100a,code=sm_100a`` only
(no PTX fallback, no other architectures) with ``-lineinfo`` so ncu source
pages map back to the .cu files.  The library links the CUDA runtime
statically and exports exactly the ``extern "C"`` symbols of include/sccg.h.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libsccg.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(INCLUDE, "sccg.h"), __file__]


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in _deps())


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None, out: str | None = None) -> str:
    """Compile csrc/*.cu for sm_100a and link libsccg.so (or `out`, an
    experiment variant built with `extra` nvcc flags).  Returns its path."""
    lib = out or LIB
    if not force and not _stale(lib):
        return lib
    bdir = BUILD if out is None else BUILD + "_" + os.path.basename(out).replace(".so", "")
    os.makedirs(bdir, exist_ok=True)
    extra = list(extra or [])

    def compile_one(src):
        obj = os.path.join(bdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", INCLUDE, "-I", CSRC, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl",
           "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python build.py [--force] [--variant NAME -DFLAG ...]
    args = sys.argv[1:]
    if "--variant" in args:
        i = args.index("--variant")
        name = args[i + 1]
        flags = [a for a in args[i + 2:]]
        print(build(force=True, verbose=True, extra=flags, out=os.path.join(PKG, f"libsccg_{name}.so")))
    else:
        print(build(force="--force" in args, verbose=True))
