"""Build the sm_100a CUDA library ``libcgs_b200.so`` in-tree with nvcc.

Each ``csrc/*.cu`` is compiled separately (in parallel) for
``-gencode arch=compute_100a,code=sm_100a`` and linked into one shared
library exporting the C ABI of ``include/cgs_b200.h``.  The CUDA runtime is
linked statically, so the library needs only the driver at run time.
Rebuilds only when a source or header is newer than the library.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libcgs_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# host code keeps each floating-point operation separately rounded (the MCMC
# host loop reproduces numpy's float expressions bit for bit)
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr", "-I", INCLUDE]


def _npyrandom() -> str:
    """numpy's own distributions library (random_normal, as Generator.normal
    runs it), linked statically for the MCMC host loop (mcmc_host.cu)."""
    import numpy
    p = os.path.join(os.path.dirname(numpy.__file__), "random", "lib", "libnpyrandom.a")
    if not os.path.exists(p):
        raise RuntimeError(f"numpy's libnpyrandom.a not found at {p}")
    return p


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(INCLUDE, "cgs_b200.h"))
    return files


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _deps() + [__file__])


def build(force: bool = False, verbose: bool = False, defines=None, out: str = None) -> str:
    """Build LIB (or, for tuning experiments, a variant with extra -D defines
    into ``out``; load it with CGS_LIB_PATH=out)."""
    lib = out or LIB
    if not force and out is None and not _stale():
        return LIB
    bdir = BUILD if out is None else out + ".objs"
    os.makedirs(bdir, exist_ok=True)
    nvcc = _nvcc()
    dflags = [f"-D{d}" for d in (defines or [])]

    def compile_one(src):
        obj = os.path.join(bdir, os.path.basename(src)[:-3] + ".o")
        cmd = [nvcc, *ARCH, *FLAGS, *dflags, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stderr.strip() or r.stdout.strip()):
            print(r.stderr, r.stdout, file=sys.stderr)
        return obj

    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = lib + ".tmp"
    # the static numpy library's symbols stay local to this .so
    cmd = [nvcc, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-Xlinker", "--exclude-libs,ALL", "-o", tmp,
           *objs, _npyrandom()]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
