"""ORACLE — test infrastructure only (the checker, never the product).

Python face of the CPU restatement of the reference SpMV path:
  * ctypes wrappers over oracle/lw_oracle.c (built by build() below into
    oracle/_build/liblworacle.so), fp64 / int64 like the reference;
  * tiny pure-Python restatements used to cross-check the C code itself
    (merge_walk_coords mirrors the reference test oracle, tests/conftest.py:40-54).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline/reference leg
may import this module. The package paper_2301_04792_b200 never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
LIB = BUILD / "liblworacle.so"
SRC = HERE / "lw_oracle.c"

_lib = None

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_int = ctypes.c_int


def build(force: bool = False) -> Path:
    """gcc -O3 -fopenmp the oracle into oracle/_build/liblworacle.so."""
    if not force and LIB.exists() and LIB.stat().st_mtime >= max(
            SRC.stat().st_mtime, (HERE.parent / "include" / "lw_hash.h").stat().st_mtime):
        return LIB
    BUILD.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
                    "-fvisibility=hidden", "-o", str(tmp), str(SRC)], check=True)
    os.replace(tmp, LIB)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB))
        sig = {
            "lwo_version": (_int, []),
            "lwo_merge_path_search": (_i64, [_p, _i64, _i64, _i64]),
            "lwo_merge_path_partition": (None, [_p, _i64, _i64, _i64, _p, _int]),
            "lwo_spmv_thread_mapped": (None, [_p, _p, _p, _p, _p, _i64, _i64, _int]),
            "lwo_spmv_merge_path": (_int, [_p, _p, _p, _p, _p, _i64, _i64, _i64, _int, _p]),
            "lwo_spmv_group_mapped": (None, [_p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _int]),
            "lwo_spmm_thread_mapped": (None, [_p, _p, _p, _p, _p, _i64, _i64, _i64, _int]),
            "lwo_spmm_merge_path": (_int, [_p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _int]),
            "lwo_spmm_group_mapped": (None, [_p, _p, _p, _p, _p, _i64, _i64, _i64, _i64, _i64,
                                             _int]),
            "lwo_sssp": (_i64, [_p, _p, _p, _i64, _i64, _p]),
            "lwo_bfs": (_i64, [_p, _p, _i64, _i64, _p]),
            "lwo_assign_thread_mapped": (None, [_p, _i64, _i64, _p, _p, _p]),
            "lwo_assign_merge_path": (None, [_p, _i64, _i64, _i64, _p, _p, _p]),
            "lwo_assign_group_mapped": (None, [_p, _i64, _i64, _i64, _i64, _p, _p, _p]),
            "lwo_rmat_keys": (None, [_int, _i64, _i64, _u32, _u32, _u32, _u64, _p, _int]),
            "lwo_hash_values": (None, [_p, _i64, _u64, _p, _int]),
            "lwo_uniform_keys": (None, [_i64, _i64, _i64, _u64, _p, _int]),
            "lwo_rmat_csr": (_i64, [_int, _i64, _u32, _u32, _u32, _u64, _int, _p, _p, _p]),
            "lwo_tolerance_f32": (ctypes.c_double, [_p, _p, _p, _i64, ctypes.c_double, _p, _int]),
            "lwo_tolerance_f64": (ctypes.c_double, [_p, _p, _p, _i64, ctypes.c_double, _p, _int]),
        }
        for ob in (32, 64):
            for vb in (32, 64):
                sig[f"lwo_spmv_narrow_o{ob}_f{vb}"] = (_int, [_p, _p, _p, _p, _p, _p, _i64, _i64, _int])
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def _i64a(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64a(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


# ---- schedules -----------------------------------------------------------------------

def merge_path_search(off, diagonal: int) -> tuple[int, int]:
    off = _i64a(off)
    rows, nnz = off.size - 1, int(off[-1])
    if not 0 <= diagonal <= rows + nnz:
        raise ValueError("diagonal out of range")
    t = lib().lwo_merge_path_search(_ptr(off), rows, nnz, diagonal)
    return int(t), int(diagonal - t)


def merge_path_partition(off, lanes: int, threads: int = 1) -> np.ndarray:
    off = _i64a(off)
    out = np.empty((lanes + 1, 2), dtype=np.int64)
    lib().lwo_merge_path_partition(_ptr(off), off.size - 1, int(off[-1]), lanes, _ptr(out), threads)
    return out


def merge_walk_coords(off) -> list[tuple[int, int]]:
    """Brute-force walk of the whole path (boundary before atom on ties)."""
    off = [int(v) for v in off]
    n_t, n_a = len(off) - 1, off[-1]
    tile = atom = 0
    out = [(0, 0)]
    for _ in range(n_t + n_a):
        if tile < n_t and off[tile + 1] <= atom:
            tile += 1
        else:
            atom += 1
        out.append((tile, atom))
    return out


def assignment(off, schedule: str, lanes: int, group_size: int = 32,
               tiles_per_block: int | None = None):
    """(lane_atoms[lanes], atom_lane[nnz], atom_tile[nnz]) for a schedule."""
    off = _i64a(off)
    rows, nnz = off.size - 1, int(off[-1])
    la = np.zeros(lanes, dtype=np.int64)
    al = np.full(max(nnz, 1), -1, dtype=np.int32)
    at = np.full(max(nnz, 1), -1, dtype=np.int32)
    L = lib()
    if schedule == "thread-mapped":
        L.lwo_assign_thread_mapped(_ptr(off), rows, lanes, _ptr(la), _ptr(al), _ptr(at))
    elif schedule == "merge-path":
        L.lwo_assign_merge_path(_ptr(off), rows, nnz, lanes, _ptr(la), _ptr(al), _ptr(at))
    elif schedule == "group-mapped":
        tpb = tiles_per_block or group_size
        L.lwo_assign_group_mapped(_ptr(off), rows, lanes, group_size, tpb, _ptr(la), _ptr(al),
                                  _ptr(at))
    else:
        raise ValueError(schedule)
    return la, al[:nnz], at[:nnz]


# ---- SpMV ----------------------------------------------------------------------------

def spmv(off, col, val, x, schedule: str = "merge-path", lanes: int | None = None,
         threads: int = 1, group_size: int = 32, tiles_per_block: int | None = None) -> np.ndarray:
    """fp64 y = A x under a schedule with the reference's lane/thread semantics."""
    off, col, val, x = _i64a(off), _i64a(col), _f64a(val), _f64a(x)
    rows, nnz = off.size - 1, int(off[-1])
    lanes = lanes or threads * 32
    y = np.zeros(rows, dtype=np.float64)
    L = lib()
    if schedule == "thread-mapped":
        L.lwo_spmv_thread_mapped(_ptr(off), _ptr(col), _ptr(val), _ptr(x), _ptr(y), rows, lanes,
                                 threads)
    elif schedule == "merge-path":
        rc = L.lwo_spmv_merge_path(_ptr(off), _ptr(col), _ptr(val), _ptr(x), _ptr(y), rows, nnz,
                                   lanes, threads, None)
        if rc:
            raise MemoryError("oracle merge-path allocation failed")
    elif schedule == "group-mapped":
        L.lwo_spmv_group_mapped(_ptr(off), _ptr(col), _ptr(val), _ptr(x), _ptr(y), rows, lanes,
                                group_size, tiles_per_block or group_size, threads)
    else:
        raise ValueError(schedule)
    return y


def spmm(off, col, val, B, schedule: str = "merge-path", lanes: int | None = None,
         threads: int = 1, group_size: int = 32, tiles_per_block: int | None = None) -> np.ndarray:
    """fp64 C = A B (B row-major [cols, n]) under a schedule, reference lane semantics
    (reference kernels.py:129-175, _fast.py:80-144)."""
    off, col, B = _i64a(off), _i64a(col), _f64a(B)
    val = _f64a(val)
    if B.ndim != 2:
        raise ValueError("B must be 2-D")
    rows, nnz, n = off.size - 1, int(off[-1]), B.shape[1]
    lanes = lanes or threads * 32
    C = np.zeros((rows, n), dtype=np.float64)
    L = lib()
    if schedule == "thread-mapped":
        L.lwo_spmm_thread_mapped(_ptr(off), _ptr(col), _ptr(val), _ptr(B), _ptr(C), rows, n, lanes,
                                 threads)
    elif schedule == "merge-path":
        if L.lwo_spmm_merge_path(_ptr(off), _ptr(col), _ptr(val), _ptr(B), _ptr(C), rows, nnz, n,
                                 lanes, threads):
            raise MemoryError("oracle spmm allocation failed")
    elif schedule == "group-mapped":
        L.lwo_spmm_group_mapped(_ptr(off), _ptr(col), _ptr(val), _ptr(B), _ptr(C), rows, n, lanes,
                                group_size, tiles_per_block or group_size, threads)
    else:
        raise ValueError(schedule)
    return C


def abs_spmm_sums(off, col, val, B) -> np.ndarray:
    """sum_j |A_ij B_jc| per (row, column) — the tolerance scale for SpMM."""
    off, col = _i64a(off), _i64a(col)
    prod = np.abs(_f64a(val)[:, None] * _f64a(B)[col])
    csum = np.concatenate([np.zeros((1, prod.shape[1])), np.cumsum(prod, axis=0)])
    return csum[off[1:]] - csum[off[:-1]]


def sssp(off, col, w, source: int) -> np.ndarray:
    """Frontier-pass SSSP exactly as the reference's numba path runs it."""
    off, col, w = _i64a(off), _i64a(col), _f64a(w)
    n = off.size - 1
    dist = np.empty(n, dtype=np.float64)
    if lib().lwo_sssp(_ptr(off), _ptr(col), _ptr(w), n, source, _ptr(dist)) < 0:
        raise MemoryError("oracle sssp allocation failed")
    return dist


def bfs(off, col, source: int) -> np.ndarray:
    off, col = _i64a(off), _i64a(col)
    n = off.size - 1
    depth = np.empty(n, dtype=np.int64)
    if lib().lwo_bfs(_ptr(off), _ptr(col), n, source, _ptr(depth)) < 0:
        raise MemoryError("oracle bfs allocation failed")
    return depth


def spmv_narrow(off, col, val, x, lanes: int | None = None, threads: int | None = None):
    """Merge-path y = A x (fp64 arithmetic, reference lanes + serial fix-up) on the
    device layout as copied back from the GPU — offsets int32/int64, columns int32,
    values and x float32/float64, widened element by element (lw_oracle.c
    LWO_NARROW_SPMV). Returns (y_ref, scale) with scale = sum_j |A_ij x_j|."""
    off = np.ascontiguousarray(off)
    col = np.ascontiguousarray(col, dtype=np.int32)
    val = np.ascontiguousarray(val)
    if off.dtype not in (np.int32, np.int64) or val.dtype not in (np.float32, np.float64):
        raise TypeError("offsets int32/int64, values float32/float64")
    x = np.ascontiguousarray(x, dtype=val.dtype)
    rows = off.size - 1
    threads = threads or default_threads()
    lanes = lanes or 32 * threads
    y = np.empty(rows, dtype=np.float64)
    scale = np.empty(rows, dtype=np.float64)
    fn = getattr(lib(), f"lwo_spmv_narrow_o{off.itemsize * 8}_f{val.itemsize * 8}")
    if fn(_ptr(off), _ptr(col), _ptr(val), _ptr(x), _ptr(y), _ptr(scale), rows, lanes, threads):
        raise MemoryError("oracle narrow spmv allocation failed")
    return y, scale


def worst_ratio(y, y_ref, scale, rtol: float, threads: int | None = None) -> tuple[float, int]:
    """max_r |y[r] - y_ref[r]| / (rtol * scale[r]) (<= 1 passes) and its row."""
    y = np.ascontiguousarray(y)
    if y.dtype not in (np.float32, np.float64):
        y = y.astype(np.float64)
    wr = ctypes.c_int64(-1)
    fn = lib().lwo_tolerance_f32 if y.dtype == np.float32 else lib().lwo_tolerance_f64
    w = fn(_ptr(y), _ptr(y_ref), _ptr(scale), y.size, rtol, ctypes.byref(wr),
           threads or default_threads())
    return float(w), int(wr.value)


def abs_row_sums(off, col, val, x) -> np.ndarray:
    """sum_j |A_ij x_j| per row — the scale of the north star's tolerance."""
    off, col = _i64a(off), _i64a(col)
    prod = np.abs(_f64a(val) * _f64a(x)[col])
    csum = np.concatenate([[0.0], np.cumsum(prod)])
    return csum[off[1:]] - csum[off[:-1]]


def tolerance_ok(y, y_ref, scale, rtol: float) -> tuple[bool, float]:
    """|y - y_ref| <= rtol * scale (+ a denormal floor); returns (ok, worst ratio)."""
    err = np.abs(np.asarray(y, dtype=np.float64) - y_ref)
    bound = rtol * np.asarray(scale) + 1e-300
    worst = float((err / np.maximum(bound, 1e-300)).max()) if err.size else 0.0
    return bool(np.all(err <= bound)), worst


# ---- inputs ---------------------------------------------------------------------------

def rmat_keys(scale: int, n_edges: int, seed: int, thresholds, edge_begin: int = 0,
              threads: int | None = None) -> np.ndarray:
    out = np.empty(n_edges, dtype=np.int64)
    ta, tab, tabc = thresholds
    lib().lwo_rmat_keys(scale, edge_begin, n_edges, ta, tab, tabc, seed, _ptr(out),
                        threads or default_threads())
    return out


def uniform_csr(rows: int, cols: int, nnz_target: int, seed: int, threads: int | None = None):
    """Host twin of device.generate_uniform_device: (off, col, val) int64/int64/fp64."""
    keys = np.empty(nnz_target, dtype=np.int64)
    lib().lwo_uniform_keys(rows * cols, 0, nnz_target, seed, _ptr(keys), threads or default_threads())
    keys = np.unique(keys)
    val = np.empty(keys.size, dtype=np.float64)
    lib().lwo_hash_values(_ptr(keys), keys.size, seed, _ptr(val), threads or default_threads())
    r = keys // cols
    off = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=rows), out=off[1:])
    return off, keys - r * cols, val


def rmat_csr(scale: int, edge_factor: int, seed: int, thresholds, threads: int | None = None):
    """(off int64[n+1], col int64[nnz], val float64[nnz]) — same matrix as the device."""
    n = 1 << scale
    cap = edge_factor * n
    off = np.empty(n + 1, dtype=np.int64)
    col = np.empty(cap, dtype=np.int64)
    val = np.empty(cap, dtype=np.float64)
    ta, tab, tabc = thresholds
    nnz = lib().lwo_rmat_csr(scale, edge_factor, ta, tab, tabc, seed, threads or default_threads(),
                             _ptr(off), _ptr(col), _ptr(val))
    if nnz < 0:
        raise MemoryError("oracle rmat allocation failed")
    return off, col[:nnz], val[:nnz]
