"""Build the CUDA library in-tree: paper_1612_04082_b200/lib/libelastobem.so (sm_100a)."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libelastobem.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-ftz=true", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def _needs(obj: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defs=(), variant: str = "") -> str:
    """Compile every csrc/*.cu and link lib/libelastobem.so.  `defs` (-D flags) with a
    `variant` name build an A/B variant instead: lib/variants/<variant>.so, selected at import
    by EBEM_LIB_VARIANT=<variant> (measurement only; the product library is the default)."""
    global OBJ, LIB
    obj_dir, lib_path = OBJ, LIB
    if variant:
        OBJ = os.path.join(PKG, "build", "variants", variant)
        LIB = os.path.join(LIBDIR, "variants", variant + ".so")
    try:
        return _build(force, verbose, [f"-D{d}" for d in defs])
    finally:
        OBJ, LIB = obj_dir, lib_path


def _build(force, verbose, dflags) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(PKG, "..", "include", "elastobem.h")]
    jobs = []
    for src in srcs:
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        if force or _needs(obj, [src, __file__] + headers):
            jobs.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [NVCC, *ARCH, *FLAGS, *dflags, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for msg in ex.map(compile_one, jobs):
            if verbose and msg:
                print(msg)
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in srcs]
    if force or jobs or not os.path.exists(LIB):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart_static", "-lrt", "-lpthread", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    import sys
    a = [x for x in sys.argv[1:] if x != "--force"]
    # python _build.py [--force] [variant DEF=1 DEF2=3 ...]
    print(build(force="--force" in sys.argv, verbose=True, variant=a[0] if a else "", defs=a[1:]))
