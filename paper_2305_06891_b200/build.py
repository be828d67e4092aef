"""Build libhm.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2305_06891_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libhm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off", "-I", CSRC,
          "-I", os.path.join(os.path.dirname(HERE), "include")]
# experiment-only engine geometry overrides (e.g. HM_BUILD_DEFINES="HM_PSTAGES=4 HM_STAGE_DOUBLES=5120")
COMMON += ["-D" + d for d in os.environ.get("HM_BUILD_DEFINES", "").split()]
# the host H-arithmetic (stage B) is vectorised, FMA-contracted and OpenMP-tasked; its results are
# compared with tolerances, so contraction is allowed there (reading R22)
EXTRA = {"hla.cpp": ["-Xcompiler", "-fopenmp,-ffp-contract=fast,-march=x86-64-v3,-mtune=sapphirerapids"]}
SOURCES = ["tree.cpp", "hop.cpp", "api.cpp", "hlu.cpp", "hla.cpp", "engine.cpp", "shard.cpp",
           "kernels_assembly.cu", "kernels_apply.cu", "kernels_dense.cu", "kernels_engine.cu",
           "kernels_mrhs.cu", "kernels_recompress.cu"]


def _digest(extra=()) -> str:
    h = hashlib.sha256()
    for f in sorted(os.listdir(CSRC)) + ["../../include/hm.h"]:
        p = os.path.join(CSRC, f)
        if os.path.isfile(p):
            h.update(f.encode())
            h.update(open(p, "rb").read())
    h.update(" ".join(ARCH + COMMON + [str(EXTRA)] + list(extra)).encode())
    return h.hexdigest()


def build(verbose: bool = False, force: bool = False, defines=(), lib: str = LIB) -> str:
    """Compile every source for sm_100a and link `lib`.  `defines`: extra -D flags (e.g. the device-check
    build, ("HM_DEVICE_CHECKS=1",), linked to another path so the product library is untouched)."""
    extra = ["-D" + d for d in defines]
    bdir = BUILD if lib == LIB else os.path.join(BUILD, os.path.splitext(os.path.basename(lib))[0])
    os.makedirs(bdir, exist_ok=True)
    stamp = os.path.join(bdir, "stamp")
    dg = _digest(extra)
    if not force and os.path.exists(lib) and os.path.exists(stamp) and open(stamp).read() == dg:
        return lib

    def compile_one(src):
        obj = os.path.join(bdir, src + ".o")
        cmd = [NVCC] + ARCH + COMMON + extra + EXTRA.get(src, []) + (["-Xptxas", "-v"] if verbose and src.endswith(".cu") else [])
        if src.endswith(".cpp"):
            cmd += ["-x", "cu"] if False else []
        cmd += ["-c", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = lib + ".tmp"
    cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-Xlinker", "--no-undefined", "-o", tmp] + objs + ["-ldl", "-lgomp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    with open(stamp, "w") as f:
        f.write(dg)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
