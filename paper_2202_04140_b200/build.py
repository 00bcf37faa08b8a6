"""Build the in-tree CUDA library libacedag_b200.so for sm_100a with nvcc.

Each translation unit compiles to an object in parallel (build/), then nvcc
links the shared library."""

from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libacedag_b200.so")
OBJ = os.path.join(HERE, "build")
SOURCES = ["capi.cu", "horner.cu", "graph.cpp", "graph_io.cpp", "plan.cpp"]
HEADERS = ["graph.h", "plan.h", "kernels.cuh", "pool.cuh", "ylm_norms.h", "horner.h"]
# headers each translation unit includes (object rebuilt when one is newer)
DEPS = {"capi.cu": HEADERS, "horner.cu": ["horner.h", "plan.h", "graph.h"],
        "graph.cpp": ["graph.h"], "graph_io.cpp": ["graph.h"], "plan.cpp": ["plan.h", "graph.h"]}
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [*GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-diag-suppress", "550"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(HERE, "..", "include", "acedag_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _obj(src: str) -> str:
    return os.path.join(OBJ, os.path.splitext(src)[0] + ".o")


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    os.makedirs(OBJ, exist_ok=True)

    def compile_one(src: str) -> None:
        extra = os.environ.get("ACEDAG_NVCC_EXTRA", "").split()  # experiment builds only
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", "-o", _obj(src), os.path.join(CSRC, src)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)

    def obj_stale(src: str) -> bool:
        o = _obj(src)
        if force or not os.path.exists(o):
            return True
        deps = [src, *DEPS.get(src, HEADERS)]
        deps = [os.path.join(CSRC, d) for d in deps] + [os.path.join(HERE, "..", "include", "acedag_b200.h")]
        return any(os.path.getmtime(d) > os.path.getmtime(o) for d in deps if os.path.exists(d))

    todo = [s for s in SOURCES if obj_stale(s)]
    with ThreadPoolExecutor(max(1, len(todo))) as ex:
        list(ex.map(compile_one, todo))
    cmd = [nvcc, *GENCODE, "-shared", "-o", OUT, *[_obj(s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
