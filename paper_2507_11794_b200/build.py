"""Build the sm_100a shared library `_lib/libclothsim_b200.so` with nvcc.

    python -m paper_2507_11794_b200.build

The library is built in-tree so it travels with the repository snapshot to
the GPU box.  Flags: -gencode arch=compute_100a,code=sm_100a (B200 only),
-O3, -lineinfo (ncu source view), no fast-math (the reference-exact modes
rely on IEEE round-to-nearest intrinsics).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libclothsim_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
SOURCES = ["cs_api.cu", "cs_grid.cu", "cs_strip.cu", "cs_pair3.cu", "cs_csr.cu", "cs_collide.cu",
           "cs_collide64.cu", "cs_snapshot.cu", "cs_gridgen.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build the extension")


def _inputs():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    files.append(os.path.join(INCLUDE, "clothsim_b200.h"))
    return files


def up_to_date() -> bool:
    if not os.path.exists(LIB_PATH):
        return False
    t = os.path.getmtime(LIB_PATH)
    return all(os.path.getmtime(f) <= t for f in _inputs())


def build(force: bool = False, verbose: bool = False, extra_flags=(), out: str | None = None) -> str:
    """Compile every translation unit in parallel (one nvcc per file), then
    link the shared library; `extra_flags` / `out` serve A/B variants."""
    from concurrent.futures import ThreadPoolExecutor

    out = out or LIB_PATH
    if not force and out == LIB_PATH and up_to_date():
        return LIB_PATH
    os.makedirs(LIB_DIR, exist_ok=True)
    objdir = os.path.join(LIB_DIR, "obj" + ("" if out == LIB_PATH else "_" + os.path.basename(out)))
    os.makedirs(objdir, exist_ok=True)
    base = [nvcc_path(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-I",
            INCLUDE, *extra_flags]
    if verbose:
        base.insert(1, "-Xptxas=-v")

    def compile_one(src):
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        cmd = base + ["-c", "-o", obj, os.path.join(CSRC, src)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src} ({res.returncode}):\n{res.stdout}\n{res.stderr}")
        if verbose:
            print(res.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = out + ".tmp"
    res = subprocess.run([nvcc_path(), *ARCH, "-shared", "-o", tmp, *objs], capture_output=True,
                         text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
