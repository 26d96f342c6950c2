"""In-tree build of the CUDA engine (libirkg.so) for sm_100a.

``python -m paper_2101_01776_b200._build`` or ``__graft_entry__.build()``.
The shared library lands next to this file so it travels with the repo
snapshot to the GPU box (built artefacts are git-ignored, not gpurun-ignored).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libirkg.so")
#: checked build: the same sources with -DIRKG_CHECKED (device bounds /
#: invariant checks that trap; the compute-sanitizer stand-in)
LIB_CHECKED = os.path.join(HERE, "libirkg_checked.so")
SOURCES = ["kernels.cu", "cgs.cu", "stencil.cu", "jacobi.cu", "jacobi3d.cu", "dae.cu", "arachain.cu", "comm.cu", "dirk.cu", "banded.cu", "mg.cu", "rcgmres.cu", "engine.cu"]
HEADERS = ["kinds.cuh", "kernels.cuh", "engine.h", os.path.join("..", "..", "include", "irkg.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
         "-Xptxas", "-v"]


HASH_FILE = LIB + ".srchash"


def source_hash():
    """Content hash of the CUDA sources + build flags (mtime-free, so it
    survives the repo snapshot to the GPU box)."""
    import hashlib

    h = hashlib.sha256()
    for f in SOURCES + HEADERS:
        with open(os.path.join(CSRC, f), "rb") as fh:
            h.update(fh.read())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def is_fresh():
    if not os.path.exists(LIB) or not os.path.exists(HASH_FILE):
        return False
    with open(HASH_FILE) as fh:
        return fh.read().strip() == source_hash()


def _stale():
    return not is_fresh()


def build(force=False, verbose=False, checked=False):
    if checked:
        return _build_into(LIB_CHECKED, ["-DIRKG_CHECKED"], "_checked", verbose)
    if not force and not _stale():
        return LIB
    return _build_into(LIB, [], "", verbose, write_hash=True)


def _build_into(lib, extra, suffix, verbose, write_hash=False):
    from concurrent.futures import ThreadPoolExecutor

    def compile_one(src):
        obj = os.path.join(CSRC, src.replace(".cu", suffix + ".o"))
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        for src, obj, res in ex.map(compile_one, SOURCES):
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(res.stderr)
            objs.append(obj)
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-L/usr/local/cuda/lib64", "-lcufft", "-Xlinker", "-rpath=/usr/local/cuda/lib64",
           "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, lib)
    if write_hash:
        with open(HASH_FILE, "w") as fh:
            fh.write(source_hash())
    return lib


if __name__ == "__main__":
    checked = "--checked" in sys.argv
    print(build(force="--force" in sys.argv, verbose=not checked, checked=checked))
