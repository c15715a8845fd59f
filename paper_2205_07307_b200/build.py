"""Build the CUDA path in-tree: paper_2205_07307_b200/libodf.so (sm_100a).

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, no fast-math/FTZ
(comparisons must be exact IEEE fp32).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libodf.so")
# one kernel family per translation unit (odf_kernels.cuh holds the templates), so
# the objects compile in parallel
SOURCES = ["odf_capi.cu", "odf_k_fused_nf.cu", "odf_k_fused_nu.cu", "odf_k_fused_wf.cu",
           "odf_k_fused_wu.cu", "odf_k_apply.cu", "odf_k_halves.cu", "odf_k_t64_f.cu", "odf_k_t64_u.cu", "odf_k_lat_u.cu",
           "odf_k_aux.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "odf.h"),
                                                                 os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile_link(out: str, defines=(), verbose: bool = False) -> None:
    """nvcc -c of every source in parallel (they are independent), then one link.
    Objects are cached under build/obj/, keyed by the flags and the bytes of the
    source and headers."""
    import hashlib
    from concurrent.futures import ThreadPoolExecutor
    common = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xfatbin", "-compress-all",
              "-Xcompiler", "-fPIC",
              "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"),
              *[f"-D{d}" for d in defines]]
    objdir = os.path.join(ROOT, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    headers = sorted([os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] +
                     [os.path.join(ROOT, "include", "odf.h")])

    def key(src):  # flags + the bytes of the source and every header it may include
        h = hashlib.sha1(" ".join(common).encode())
        for f in [src, *headers]:
            with open(f, "rb") as fh:
                h.update(fh.read())
        return h.hexdigest()[:16]

    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    objs = [os.path.join(objdir, f"{os.path.splitext(s)[0]}.{key(p)}.o") for s, p in zip(SOURCES, srcs)]

    def cc(i):
        if os.path.exists(objs[i]) and not verbose:
            return
        tmp = objs[i] + f".tmp{os.getpid()}"
        subprocess.check_call([*common, "-Xptxas", "-v" if verbose else "-O3", "-c", srcs[i], "-o", tmp])
        os.replace(tmp, objs[i])

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        list(ex.map(cc, range(len(SOURCES))))
    subprocess.check_call([nvcc(), *ARCH, "-shared", *objs, "-o", out, "-ldl"])


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    _compile_link(tmp, verbose=verbose)
    os.replace(tmp, LIB)
    return LIB


def build_variant(out: str, defines=()) -> str:
    """Diagnostics / A-B builds (tools only, loaded via ODF_LIB_OVERRIDE): same sources
    with extra -D flags, written to `out`.  The product library is build()'s."""
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    _compile_link(out, defines)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
