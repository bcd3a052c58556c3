"""Build liblwb200.so (the sm_100a kernels + C ABI) in-tree with nvcc.

The library is a plain shared object with an ``extern "C"`` surface
(include/lw_b200.h), loaded by ctypes; no torch headers are involved, so the
same .so serves the Python package, the bench and any FFI binding
(INTEGRATION.md). Output: paper_2301_04792_b200/_lib/liblwb200.so.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "liblwb200.so"
STAMP = LIBDIR / "liblwb200.stamp"

SOURCES = [
    "lw_abi.cu",
    "spmv_thread_mapped.cu",
    "spmv_work_oriented.cu",
    "hotx.cu",
    "spmv_group_mapped.cu",
    "spmm.cu",
    "frontier.cu",
    "vector_ops.cu",
    "generators.cu",
    "mmio.cpp",
]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; set NVCC or put /usr/local/cuda/bin on PATH")


def _digest() -> str:
    h = hashlib.sha256()
    for p in sorted(list(CSRC.glob("*")) + list(INCLUDE.glob("*.h")) + [Path(__file__)]):
        if p.is_file():
            h.update(p.name.encode())
            h.update(p.read_bytes())
    h.update(" ".join(ARCH + FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile every .cu into liblwb200.so unless the sources are unchanged."""
    digest = _digest()
    if not force and LIB.exists() and STAMP.exists() and STAMP.read_text() == digest:
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    nvcc = _nvcc()
    objdir = LIBDIR / "obj"
    objdir.mkdir(exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc, *ARCH, *FLAGS, "-I", str(INCLUDE), "-I", str(CSRC), "-c", str(CSRC / src),
               "-o", str(obj)]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(str(obj))
    for cmd, proc in procs:
        out, _ = proc.communicate()
        if proc.returncode != 0 or verbose:
            sys.stderr.write(out.decode(errors="replace"))
        if proc.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    tmp = LIB.with_suffix(".so.tmp")
    link = [nvcc, *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart"]
    subprocess.run(link, check=True)
    os.replace(tmp, LIB)
    STAMP.write_text(digest)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
