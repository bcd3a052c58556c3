"""Host CSR container, validation and synthetic generators.

``CsrMatrix`` mirrors the reference container (sparse.py:40-71): int64 offsets
and column indices, float64 values, so a reference user's matrices drop in
unchanged. Device storage (int32 indices, fp32/fp64 values) lives in
:class:`~paper_2301_04792_b200.device.DeviceCsr`.

Generators:
  * ``generate_random_csr`` / ``generate_power_law_csr`` reproduce the
    reference generators (sparse.py:164-223) draw for draw, so identical seeds
    give identical matrices (pinned by tests/golden). The power-law one draws
    all row samples in one call instead of one call per row — NumPy's
    Generator yields the same stream either way — and de-duplicates with one
    sort, so 2^20-row matrices build in seconds instead of ~20 s.
  * ``generate_banded_csr`` and ``generate_rmat_csr`` are new (the north star's
    C2b/C3/C5 inputs). Their values/keys are counter-based hashes
    (include/lw_hash.h), identical on the device generator and the C oracle.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["CooMatrix", "CsrMatrix", "Graph", "validate_coo", "validate_csr", "coo_to_csr",
           "csr_to_coo", "transpose_csr", "generate_random_csr", "generate_power_law_csr",
           "generate_banded_csr", "rmat_thresholds", "hash_values_np", "row_length_stats"]

MASK64 = (1 << 64) - 1


@dataclass
class CsrMatrix:
    """Compressed sparse rows; offsets start at 0, end at nnz, never decrease."""

    rows: int
    cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.rows = int(self.rows)
        self.cols = int(self.cols)
        self.row_offsets = np.ascontiguousarray(self.row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(self.col_indices, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)

    @property
    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    def row_lengths(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols))
        r = np.repeat(np.arange(self.rows), self.row_lengths())
        out[r, self.col_indices] = self.values
        return out

    def to_device(self, dtype="float32", device=None, offset_bits: int | None = None):
        """Upload to the GPU as a DeviceCsr (int32 col_idx, fp32/fp64 values)."""
        from .device import DeviceCsr

        return DeviceCsr.from_host(self, dtype=dtype, device=device, offset_bits=offset_bits)


@dataclass
class CooMatrix:
    """Coordinate-format matrix; entries may be unsorted and may repeat (reference
    sparse.py:14-37)."""

    rows: int
    cols: int
    row: np.ndarray
    col: np.ndarray
    data: np.ndarray

    def __post_init__(self):
        self.row = np.asarray(self.row, dtype=np.int64)
        self.col = np.asarray(self.col, dtype=np.int64)
        self.data = np.asarray(self.data, dtype=np.float64)
        if not (self.row.shape == self.col.shape == self.data.shape):
            raise ValueError("row, col and data must have equal length")

    @property
    def nnz(self) -> int:
        return self.row.size

    def entries(self):
        """Iterate (row, col, value) tuples; mainly for small-matrix tests."""
        return zip(self.row.tolist(), self.col.tolist(), self.data.tolist())


def validate_coo(m: CooMatrix) -> None:
    """Raise ValueError if any entry lies outside the declared shape (sparse.py:74-81)."""
    if m.rows < 0 or m.cols < 0:
        raise ValueError("negative dimensions")
    if m.nnz and (int(m.row.min()) < 0 or int(m.row.max()) >= m.rows or int(m.col.min()) < 0
                  or int(m.col.max()) >= m.cols):
        raise ValueError("entry index out of bounds")


def coo_to_csr(coo: CooMatrix, threads: int = 0) -> CsrMatrix:
    """Sort entries by (row, col), sum duplicates, pack CSR (reference sparse.py:130-150).

    Runs in the native library (lw_coo_to_csr_host: multi-threaded sort, then
    duplicates summed in input order, exactly as lexsort + bincount do)."""
    import ctypes

    from . import _lib

    validate_coo(coo)
    n = coo.nnz
    row = np.ascontiguousarray(coo.row, dtype=np.int64)
    col = np.ascontiguousarray(coo.col, dtype=np.int64)
    data = np.ascontiguousarray(coo.data, dtype=np.float64)
    off = np.zeros(coo.rows + 1, dtype=np.int64)
    col_out = np.empty(n, dtype=np.int64)
    val_out = np.empty(n, dtype=np.float64)
    nnz = ctypes.c_int64(0)

    def ptr(a):
        return a.ctypes.data if a.size else None

    rc = _lib.load().lw_coo_to_csr_host(coo.rows, coo.cols, n, ptr(row), ptr(col), ptr(data),
                                        ptr(off), ptr(col_out), ptr(val_out), ctypes.byref(nnz),
                                        threads)
    _lib.check(rc, "coo_to_csr")
    return CsrMatrix(coo.rows, coo.cols, off, col_out[:nnz.value], val_out[:nnz.value])


def csr_to_coo(m: CsrMatrix) -> CooMatrix:
    row = np.repeat(np.arange(m.rows), m.row_lengths())
    return CooMatrix(m.rows, m.cols, row, m.col_indices.copy(), m.values.copy())


def transpose_csr(m: CsrMatrix) -> CsrMatrix:
    """Transpose via COO; the load-time answer to column-compressed inputs."""
    coo = csr_to_coo(m)
    return coo_to_csr(CooMatrix(m.cols, m.rows, coo.col, coo.row, coo.data))


class Graph:
    """A square CSR matrix read as adjacency (reference sparse.py:106-127): row =
    source vertex, nonzero = out-edge, column = neighbour, value = edge weight.
    Negative weights are rejected so shortest-path kernels can assume
    non-negativity."""

    def __init__(self, csr: CsrMatrix):
        if csr.rows != csr.cols:
            raise ValueError("adjacency matrix must be square")
        if csr.nnz and float(csr.values.min()) < 0:
            raise ValueError("edge weights must be non-negative")
        self.csr = csr

    @property
    def num_vertices(self) -> int:
        return self.csr.rows

    @property
    def num_edges(self) -> int:
        return self.csr.nnz


def validate_csr(m: CsrMatrix) -> None:
    """Raise ValueError on the first broken CSR invariant (reference sparse.py:84-103)."""
    off = m.row_offsets
    if off.shape[0] != m.rows + 1:
        raise ValueError("row_offsets must have length rows+1")
    if off[0] != 0:
        raise ValueError("row_offsets[0] must be 0")
    if off[-1] != m.nnz:
        raise ValueError("row_offsets[-1] must equal nnz")
    if m.values.shape[0] != m.nnz:
        raise ValueError("values and col_indices must have equal length")
    lengths = np.diff(off)
    if lengths.size and int(lengths.min()) < 0:
        raise ValueError("row_offsets must be nondecreasing")
    if m.nnz:
        c = m.col_indices
        if int(c.min()) < 0 or int(c.max()) >= m.cols:
            raise ValueError("column index out of bounds")
        step_ok = np.diff(c) > 0
        row_change = np.zeros(m.nnz - 1, dtype=bool)
        starts = off[1:-1]
        starts = starts[(starts > 0) & (starts < m.nnz)]
        row_change[starts - 1] = True
        if not bool(np.all(step_ok | row_change)):
            raise ValueError("column indices must be strictly increasing within a row")


def _pack(rows: int, cols: int, row_ids: np.ndarray, col_ids: np.ndarray, values) -> CsrMatrix:
    counts = np.bincount(row_ids, minlength=rows) if rows else np.zeros(0, np.int64)
    off = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return CsrMatrix(rows, cols, off, col_ids, values)


def generate_random_csr(rows: int, cols: int, nnz_target: int, seed: int) -> CsrMatrix:
    """Exactly ``nnz_target`` distinct uniform positions, values U[-1, 1].

    Same draws as the reference (sparse.py:164-187): ``choice`` without
    replacement for dense-ish shapes, rejection rounds of ``integers`` + unique +
    permutation otherwise, then sorted positions and ``uniform`` values.
    """
    cap = rows * cols
    if nnz_target > cap:
        raise ValueError(f"nnz_target {nnz_target} exceeds capacity {cap}")
    rng = np.random.default_rng(seed)
    if cap <= (1 << 22) or cap <= 4 * nnz_target:
        picked = rng.choice(cap, size=nnz_target, replace=False)
    else:
        pool = np.empty(0, dtype=np.int64)
        batch = nnz_target + nnz_target // 4 + 16
        while pool.size < nnz_target:
            pool = np.unique(np.concatenate([pool, rng.integers(0, cap, size=batch)]))
        picked = rng.permutation(pool)[:nnz_target]
    picked = np.sort(picked)
    vals = rng.uniform(-1.0, 1.0, size=nnz_target)
    if cols:
        r, c = np.divmod(picked, cols)
    else:
        r = c = picked
    return _pack(rows, cols, r, c, vals)


def generate_power_law_csr(rows: int, avg_degree: float, skew: float, seed: int) -> CsrMatrix:
    """Square matrix with truncated-Zipf row lengths (reference sparse.py:190-223).

    Row lengths: inverse-CDF draws of P(Z >= k) = k^-skew clipped to [1, rows],
    rescaled to mean ``avg_degree``; each row samples its columns uniformly
    with replacement and keeps the distinct ones; values U[-1, 1].
    """
    if rows <= 0:
        raise ValueError("rows must be positive")
    if avg_degree <= 0:
        raise ValueError("avg_degree must be positive")
    if skew <= 0:
        raise ValueError("skew must be positive")
    rng = np.random.default_rng(seed)
    raw = np.minimum(np.floor(rng.random(rows) ** (-1.0 / skew)), float(rows))
    lengths = np.minimum(np.rint(raw * (avg_degree / raw.mean())).astype(np.int64), rows)
    lengths = np.maximum(lengths, 0)
    samples = rng.integers(0, rows, size=int(lengths.sum()))
    owner = np.repeat(np.arange(rows, dtype=np.int64), lengths)
    key = owner * rows + samples
    key.sort(kind="stable")
    keep = np.ones(key.size, dtype=bool)
    keep[1:] = key[1:] != key[:-1]
    key = key[keep]
    r, c = np.divmod(key, rows)
    vals = rng.uniform(-1.0, 1.0, size=key.size)
    return _pack(rows, rows, r, c, vals)


# ---- counter-based generators (shared with the device and the C oracle) -------------

def _mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def hash_values_np(keys: np.ndarray, seed: int) -> np.ndarray:
    """NumPy twin of lw_hash_value (include/lw_hash.h): U[-1, 1) per 64-bit key."""
    with np.errstate(over="ignore"):
        s = _mix64(np.uint64((seed ^ 0x5851F42D4C957F2D) & MASK64))
        h = _mix64(s + np.asarray(keys, dtype=np.int64).astype(np.uint64) * np.uint64(0x9E3779B97F4A7C15))
    return (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0) * 2.0 - 1.0


def rmat_thresholds(a: float = 0.57, b: float = 0.19, c: float = 0.19) -> tuple[int, int, int]:
    """32-bit quadrant thresholds (t_a, t_ab, t_abc) shared by every R-MAT generator."""
    if min(a, b, c) < 0 or a + b + c > 1.0:
        raise ValueError("R-MAT probabilities must be non-negative with a+b+c <= 1")
    scale = 4294967296.0
    ta = min(int(a * scale), 0xFFFFFFFF)
    tab = min(int((a + b) * scale), 0xFFFFFFFF)
    tabc = min(int((a + b + c) * scale), 0xFFFFFFFF)
    return ta, tab, tabc


def rmat_keys_np(scale: int, n_edges: int, seed: int, thresholds) -> np.ndarray:
    """NumPy twin of lw_rmat_key for small scales (tests pin the device/C versions)."""
    ta, tab, tabc = (np.uint64(t) for t in thresholds)
    e = np.arange(n_edges, dtype=np.uint64)
    with np.errstate(over="ignore"):
        root = _mix64(_mix64(np.uint64((seed + 0x9E3779B97F4A7C15) & MASK64))
                      ^ (e * np.uint64(0xD6E8FEB86659FD93)))
        row = np.zeros(n_edges, dtype=np.uint64)
        col = np.zeros(n_edges, dtype=np.uint64)
        for level in range(scale):
            w = _mix64(root + np.uint64(level // 2 + 1) * np.uint64(0x9E3779B97F4A7C15))
            r = (w >> np.uint64(32)) if level & 1 else (w & np.uint64(0xFFFFFFFF))
            rb = (r >= tab).astype(np.uint64)
            cb = (((r >= ta) & (r < tab)) | (r >= tabc)).astype(np.uint64)
            row = (row << np.uint64(1)) | rb
            col = (col << np.uint64(1)) | cb
    return ((row << np.uint64(scale)) | col).astype(np.int64)


def rmat_csr_from_keys(scale: int, keys: np.ndarray, seed: int) -> CsrMatrix:
    """Deduplicate R-MAT keys into CSR with hashed U[-1, 1) values."""
    n = 1 << scale
    u = np.unique(keys)
    r = u >> scale
    c = u & (n - 1)
    return _pack(n, n, r, c, hash_values_np(u, seed))


def generate_banded_csr(rows: int, half_bandwidth: int, seed: int) -> CsrMatrix:
    """Square banded matrix: row i holds columns i-h .. i+h clipped to [0, rows).

    Values are hash_values_np(i*rows + j, seed). C2b is rows=1_000_000, h=16
    (32,999,728 nonzeros).
    """
    if rows <= 0 or half_bandwidth < 0:
        raise ValueError("rows must be positive and half_bandwidth non-negative")
    i = np.arange(rows, dtype=np.int64)
    lo = np.maximum(i - half_bandwidth, 0)
    hi = np.minimum(i + half_bandwidth + 1, rows)
    lengths = hi - lo
    off = np.zeros(rows + 1, dtype=np.int64)
    np.cumsum(lengths, out=off[1:])
    owner = np.repeat(i, lengths)
    cols = np.arange(off[-1], dtype=np.int64) - np.repeat(off[:-1], lengths) + np.repeat(lo, lengths)
    vals = hash_values_np(owner * rows + cols, seed)
    return CsrMatrix(rows, rows, off, cols, vals)


def row_length_stats(off: np.ndarray) -> dict:
    """Mean, std, CV and max/mean of row lengths (reported beside every sweep line)."""
    lengths = np.diff(np.asarray(off, dtype=np.int64))
    mean = float(lengths.mean()) if lengths.size else 0.0
    std = float(lengths.std()) if lengths.size else 0.0
    return {"rows": int(lengths.size), "nnz": int(lengths.sum()), "mean": mean, "std": std,
            "cv": std / mean if mean else 0.0, "max": int(lengths.max()) if lengths.size else 0,
            "max_over_mean": (float(lengths.max()) / mean) if mean else 0.0,
            "empty_rows": int((lengths == 0).sum())}
