"""Device-resident CSR and the thin launch layer over liblwb200.so.

Layout in HBM (one allocation per array, torch caching allocator):
  row_offsets  int32[rows+1] (int64 when nnz >= 2^31)
  col_indices  int32[nnz]
  values       fp32[nnz] or fp64[nnz]
x and y are dense fp32/fp64 vectors of the same dtype. Nothing is padded: the
kernels handle ragged rows and misaligned vector starts themselves.

PyTorch is plumbing here (allocation, streams, torch.distributed); every
computation goes through the C ABI in include/lw_b200.h.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["DeviceCsr", "cached_device_csr", "drop_device_cache", "device_merge_path_partition",
           "device_group_plan_prefix",
           "generate_rmat_csr", "generate_banded_device", "Workspace", "Probe", "current_stream"]


def _torch():
    import torch

    return torch


def _dtype_code(dt) -> int:
    torch = _torch()
    if dt in (torch.float32, np.float32, "float32", "f32", "fp32"):
        return _lib.LW_F32
    if dt in (torch.float64, np.float64, "float64", "f64", "fp64"):
        return _lib.LW_F64
    raise ValueError(f"unsupported value dtype {dt!r}; expected float32 or float64")


def _torch_dtype(dt):
    torch = _torch()
    return torch.float32 if _dtype_code(dt) == _lib.LW_F32 else torch.float64


def current_stream(device=None) -> int:
    torch = _torch()
    return int(torch.cuda.current_stream(device).cuda_stream)


def _require_cuda(device=None):
    torch = _torch()
    if not torch.cuda.is_available():
        raise _lib.BackendUnavailable("CUDA backend requires a visible CUDA device")
    _lib.load()
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


@dataclass
class DeviceCsr:
    """CSR matrix resident in GPU memory (the device-side tile set: rows = tiles)."""

    rows: int
    cols: int
    row_offsets: "object"   # torch int32/int64 [rows+1]
    col_indices: "object"   # torch int32 [nnz]
    values: "object"        # torch float32/float64 [nnz]

    def __post_init__(self):
        self._check()

    def _check(self) -> None:
        """The layout the kernels assume (lw_csr_t, include/lw_b200.h): raises
        ValueError instead of letting a kernel read a wrongly typed, strided or
        short array."""
        torch = _torch()
        off, col, val = self.row_offsets, self.col_indices, self.values
        for name, t in (("row_offsets", off), ("col_indices", col), ("values", val)):
            if not isinstance(t, torch.Tensor):
                raise TypeError(f"DeviceCsr.{name} must be a torch tensor")
            if t.ndim != 1 or not t.is_contiguous():
                raise ValueError(f"DeviceCsr.{name} must be a contiguous 1-D tensor")
            if t.device.type != "cuda":
                raise ValueError(f"DeviceCsr.{name} must live on a CUDA device")
        if not (off.device == col.device == val.device):
            raise ValueError("DeviceCsr tensors must share one CUDA device")
        if col.dtype != torch.int32:
            raise ValueError(f"col_indices must be int32, got {col.dtype}")
        if off.dtype not in (torch.int32, torch.int64):
            raise ValueError(f"row_offsets must be int32 or int64, got {off.dtype}")
        if val.dtype not in (torch.float32, torch.float64):
            raise ValueError(f"values must be float32 or float64, got {val.dtype}")
        if self.rows < 0 or self.cols < 0 or self.cols >= (1 << 31):
            raise ValueError("rows must be >= 0 and 0 <= cols < 2^31")
        if off.shape[0] != self.rows + 1:
            raise ValueError(f"row_offsets has {off.shape[0]} entries, expected rows+1 = {self.rows + 1}")
        if val.shape[0] != col.shape[0]:
            raise ValueError("values and col_indices differ in length")
        if off.dtype == torch.int32 and col.shape[0] >= (1 << 31):
            raise ValueError("nnz >= 2^31 needs int64 row_offsets")

    @property
    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    @property
    def device(self):
        return self.values.device

    @property
    def dtype(self):
        return self.values.dtype

    @property
    def offset_bits(self) -> int:
        return 32 if self.row_offsets.dtype == _torch().int32 else 64

    # tile-set protocol (host reads; for schedules on small matrices)
    @property
    def num_tiles(self) -> int:
        return self.rows

    @property
    def num_atoms(self) -> int:
        return self.nnz

    @property
    def offsets(self) -> np.ndarray:
        return self.row_offsets.to("cpu").numpy().astype(np.int64)

    def atom_offset(self, tile: int) -> int:
        return int(self.row_offsets[tile].item())

    @classmethod
    def from_host(cls, m, dtype="float32", device=None, offset_bits: int | None = None,
                  non_blocking: bool = False) -> "DeviceCsr":
        torch = _torch()
        dev = _require_cuda(device)
        nnz = int(m.col_indices.shape[0])
        if offset_bits is None:
            offset_bits = 32 if nnz < (1 << 31) else 64
        if offset_bits not in (32, 64) or (offset_bits == 32 and nnz >= (1 << 31)):
            raise ValueError("offset_bits must be 64 when nnz >= 2^31 (else 32 or 64)")
        if int(m.cols) >= (1 << 31):
            raise ValueError("cols must be < 2^31 (int32 column indices)")
        odt = torch.int32 if offset_bits == 32 else torch.int64
        off = torch.as_tensor(np.asarray(m.row_offsets)).to(dev, non_blocking=non_blocking).to(odt)
        col = torch.as_tensor(np.asarray(m.col_indices)).to(dev, non_blocking=non_blocking).to(torch.int32)
        val = torch.as_tensor(np.asarray(m.values)).to(dev, non_blocking=non_blocking).to(_torch_dtype(dtype))
        return cls(int(m.rows), int(m.cols), off.contiguous(), col.contiguous(), val.contiguous())

    def to_host(self):
        from .sparse import CsrMatrix

        return CsrMatrix(self.rows, self.cols, self.row_offsets.cpu().numpy(),
                         self.col_indices.cpu().numpy(), self.values.cpu().numpy())

    def astype(self, dtype) -> "DeviceCsr":
        return DeviceCsr(self.rows, self.cols, self.row_offsets, self.col_indices,
                         self.values.to(_torch_dtype(dtype)))

    def row_slice(self, r0: int, r1: int) -> "DeviceCsr":
        """Rows [r0, r1) as a CSR with rebased offsets (views, no copy of atoms)."""
        if not 0 <= r0 <= r1 <= self.rows:
            raise ValueError("row range outside the matrix")
        off = self.row_offsets[r0:r1 + 1]
        a0 = int(off[0].item())
        a1 = int(off[-1].item())
        return DeviceCsr(r1 - r0, self.cols, (off - a0).contiguous(),
                         self.col_indices[a0:a1], self.values[a0:a1])

    def c_struct(self) -> _lib.LwCsr:
        """The lw_csr_t view, cached while the three tensors are the same objects
        (held strongly, compared with ``is``) at the same ``_version`` (in-place
        edits bump it)."""
        key = self._tensor_key()
        hit = self.__dict__.get("_c_struct")
        if hit is not None and _same_key(hit[0], key):
            return hit[1]
        self._check()
        s = self._make_c_struct()
        self.__dict__["_c_struct"] = (key, s)
        return s

    def _make_c_struct(self) -> _lib.LwCsr:
        s = _lib.LwCsr()
        s.rows, s.cols, s.nnz = self.rows, self.cols, self.nnz
        s.row_offsets = self.row_offsets.data_ptr()
        s.col_indices = self.col_indices.data_ptr() if self.nnz else None
        s.values = self.values.data_ptr() if self.nnz else None
        s.offset_bits = self.offset_bits
        s.dtype = _dtype_code(self.dtype)
        return s

    # ---- hot-x column packing (csrc/hotx.cu) ----------------------
    def pack_hot_columns(self, max_hot: int | None = None) -> "HotColumns":
        """Build (once) the hot-x packing the work_oriented SpMV then uses.

        The at most ``max_hot`` most gathered columns (default 48 KB of values:
        12288 fp32 / 6144 fp64) get dense slots of a per-call packed x that the
        kernel keeps in L1; y stays bit-identical to the unpacked kernel. Costs
        one int32 copy of col_indices. Synchronizes the current stream once.
        The packing shares row_offsets / values with the matrix and follows
        tensor replacement (a new col_indices tensor drops it), but an in-place
        edit of col_indices is not seen: call drop_hot_columns() after one.
        """
        torch = _torch()
        if max_hot is None:
            max_hot = 49152 // self.values.element_size()
        max_hot = int(max_hot)
        hit = self.hot_columns()
        if hit is not None and hit.max_hot == max_hot:
            return hit
        lib = _lib.load()
        A = self.c_struct()
        col_packed = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=self.device)
        hot = torch.empty(max(max_hot, 1), dtype=torch.int32, device=self.device)
        need = lib.lw_hotx_build_workspace(self.cols)
        ws = torch.empty(max(need, 1), dtype=torch.uint8, device=self.device)
        n = ctypes.c_int32(0)
        rc = lib.lw_hotx_build(A, max_hot, col_packed.data_ptr(), hot.data_ptr(), ctypes.byref(n),
                               ws.data_ptr(), need, current_stream(self.device))
        _lib.check(rc, "lw_hotx_build")
        packed = DeviceCsr(self.rows, self.cols, self.row_offsets, col_packed[: self.nnz], self.values)
        hx = HotColumns(packed, hot[: n.value], n.value, max_hot, self._tensor_key())
        self.__dict__["_hotx"] = hx
        return hx

    def degree_relabel(self) -> "Relabeled":
        """Symmetric degree relabeling P A P^T (one-time inspector for the
        iterated SpMV, C5): vertices renumbered by decreasing in-degree (column
        count; ties by index), so the most gathered x entries form a dense
        prefix of x' = P x that stays in L2/L1, and the rows follow the same
        renumbering so y' = P y feeds the next iteration directly. Each row keeps
        its atoms in order: its products and their sequence are unchanged. The
        caller iterates on ``.matrix`` from ``P x0`` (``.to_new``) and maps the
        result back once (``.to_old``). Square matrices only."""
        torch = _torch()
        if self.rows != self.cols:
            raise ValueError("degree_relabel needs a square matrix")
        n = self.rows
        counts = torch.bincount(self.col_indices.to(torch.int64), minlength=n) if self.nnz else \
            torch.zeros(n, dtype=torch.int64, device=self.device)
        order = torch.sort(counts, descending=True, stable=True).indices      # new -> old
        rank = torch.empty(n, dtype=torch.int32, device=self.device)
        rank[order] = torch.arange(n, dtype=torch.int32, device=self.device)  # old -> new
        lengths = (self.row_offsets[1:] - self.row_offsets[:-1]).to(torch.int64)[order]
        off = torch.zeros(n + 1, dtype=torch.int64, device=self.device)
        torch.cumsum(lengths, 0, out=off[1:])
        off = off.to(self.row_offsets.dtype)
        col = torch.empty_like(self.col_indices)
        val = torch.empty_like(self.values)
        lib = _lib.load()
        _lib.check(lib.lw_csr_permute(self.c_struct(), order.data_ptr(), rank.data_ptr(), off.data_ptr(),
                                      col.data_ptr() if self.nnz else None,
                                      val.data_ptr() if self.nnz else None, current_stream(self.device)),
                   "lw_csr_permute")
        return Relabeled(DeviceCsr(n, n, off, col, val), order, rank)

    def hot_columns(self) -> "HotColumns | None":
        """The hot-x packing built by pack_hot_columns, if the tensors are unchanged."""
        hx = self.__dict__.get("_hotx")
        if hx is None:
            return None
        if not _same_key(hx.key, self._tensor_key()):
            self.__dict__.pop("_hotx", None)   # the source tensors changed: drop the packing
            return None
        return hx

    def drop_hot_columns(self) -> None:
        self.__dict__.pop("_hotx", None)

    def _tensor_key(self):
        """Strong references to the three tensors plus their versions: a cache
        entry matches only the very same tensor objects, unmodified."""
        ts = (self.row_offsets, self.col_indices, self.values)
        return (ts, tuple(t._version for t in ts), self.rows, self.cols)

    def algorithmic_bytes(self) -> int:
        """SURVEY §8(d) byte model: nnz*(idx+val) + (rows+1)*off + cols*val + rows*val."""
        sv = self.values.element_size()
        so = self.row_offsets.element_size()
        return self.nnz * (4 + sv) + (self.rows + 1) * so + self.cols * sv + self.rows * sv


def cached_device_csr(m, dtype="float64", device=None) -> "DeviceCsr":
    """Device copy of a host CsrMatrix, reused while its arrays are the same objects.

    The reference's containers are immutable by convention (reference
    sparse.py:1-7), so a host-API call (``spmv(m, x)`` with NumPy operands) need
    not re-upload the matrix every time: the DeviceCsr is kept on the matrix and
    reused while ``rows``, ``cols`` and the three arrays are unchanged. The cache
    entry holds the arrays themselves and compares them with ``is`` (an id()
    could be reused by a new array once the old one is freed), so rebinding an
    array (``m.values = ...``) always re-uploads; mutating one in place is
    outside the contract — call ``drop_device_cache(m)`` after doing so.
    """
    dev = _require_cuda(device)
    arrays = (m.row_offsets, m.col_indices, m.values)
    slot = (int(m.rows), int(m.cols), str(_torch_dtype(dtype)), str(dev))
    cache = m.__dict__.setdefault("_lw_device_cache", {})
    hit = cache.get(slot)
    if hit is not None and all(a is b for a, b in zip(hit[0], arrays)):
        return hit[1]
    d = DeviceCsr.from_host(m, dtype=dtype, device=dev)
    cache[slot] = (arrays, d)
    return d


_H2D_CHUNK = 1 << 24   # bytes per staged piece of a pipelined upload


def host_to_device(a: np.ndarray, device, dtype=None):
    """Upload a host NumPy array through pinned staging: a parallel CPU copy
    into a pinned block from torch's caching host allocator (reused across
    calls), then an async H2D DMA on the current stream — ~4x the throughput of
    a pageable copy for the host-API operands. Arrays above 16 MB go up in 16 MB
    pieces, so the CPU copy of piece i+1 overlaps the DMA of piece i (C3 fp64 x,
    128 MB: 4.6 -> ~2.9 ms). ``dtype`` converts on the device."""
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(a)).reshape(-1)
    stage = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    d = torch.empty(t.shape, dtype=t.dtype, device=device)
    step = max(1, _H2D_CHUNK // max(1, t.element_size()))
    for i in range(0, max(t.numel(), 1), step):
        stage[i:i + step].copy_(t[i:i + step])
        # async DMA; the allocator keeps `stage` alive until the copies end
        d[i:i + step].copy_(stage[i:i + step], non_blocking=True)
    d = d.reshape(a.shape)
    return d if dtype is None or d.dtype == dtype else d.to(dtype)


def device_to_host(t) -> np.ndarray:
    """Download a device tensor as float64-or-native NumPy whose storage is a
    pinned block (DMA straight into it, no pageable bounce); the array keeps
    the block alive and returns it to the cache when it is freed."""
    torch = _torch()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


def drop_device_cache(m) -> None:
    """Forget the device copies cached on a host CsrMatrix (after in-place edits)."""
    m.__dict__.pop("_lw_device_cache", None)


class Workspace:
    """Grow-only device scratch buffers, one per (device, stream), reused across
    launches: calls on one stream are ordered, so they may share a buffer; calls
    on different streams get different buffers and can run concurrently."""

    def __init__(self):
        self._buf = {}

    def get(self, nbytes: int, device, stream: int = 0):
        key = (device, stream)
        buf = self._buf.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = _torch().empty(max(nbytes, 256), dtype=_torch().uint8, device=device)
            self._buf[key] = buf
        return buf


class Probe:
    """Device buffers for the instrumented kernels (lw_probe_t)."""

    def __init__(self, lanes: int, nnz: int, device):
        torch = _torch()
        self.lane_atoms = torch.zeros(max(lanes, 1), dtype=torch.int64, device=device)
        self.atom_lane = torch.full((max(nnz, 1),), -1, dtype=torch.int32, device=device)
        self.atom_tile = torch.full((max(nnz, 1),), -1, dtype=torch.int32, device=device)
        self.atom_visits = torch.zeros(max(nnz, 1), dtype=torch.int32, device=device)
        self.lanes, self.nnz = lanes, nnz

    def c_struct(self) -> _lib.LwProbe:
        p = _lib.LwProbe()
        p.lane_atoms = self.lane_atoms.data_ptr()
        p.atom_lane = self.atom_lane.data_ptr()
        p.atom_tile = self.atom_tile.data_ptr()
        p.atom_visits = self.atom_visits.data_ptr()
        return p

    def host(self) -> dict:
        return {"lane_atoms": self.lane_atoms[: self.lanes].cpu().numpy(),
                "atom_lane": self.atom_lane[: self.nnz].cpu().numpy(),
                "atom_tile": self.atom_tile[: self.nnz].cpu().numpy(),
                "atom_visits": self.atom_visits[: self.nnz].cpu().numpy()}


@dataclass
class Relabeled:
    """A symmetric relabeling P A P^T: ``matrix`` is the permuted operator,
    ``order[i']`` the original index of new vertex i', ``rank`` its inverse."""

    matrix: DeviceCsr
    order: object
    rank: object

    def to_new(self, v):
        """P v: original numbering -> relabeled (v'[i'] = v[order[i']])."""
        return v.index_select(0, self.order)

    def to_old(self, v):
        """P^T v': relabeled numbering -> original (v[i] = v'[rank[i]])."""
        return v.index_select(0, self.rank.to(self.order.dtype))


@dataclass
class HotColumns:
    """A DeviceCsr's hot-x packing: ``packed`` is the matrix with hot columns
    relabeled to ``slot | 0x80000000`` (csrc/hotx.cu), ``hot_cols[slot]`` the
    original column of each slot (ascending), ``n_hot`` the slot count."""

    packed: DeviceCsr
    hot_cols: "object"   # torch int32 [n_hot]
    n_hot: int
    max_hot: int
    key: tuple

    def original_col_indices(self):
        """Undo the relabeling (equals the source matrix's col_indices)."""
        torch = _torch()
        c = self.packed.col_indices
        hot = c < 0
        return torch.where(hot, self.hot_cols[(c & 0x7FFFFFFF).long().clamp_(max=max(self.n_hot - 1, 0))]
                           if self.n_hot else c, c)


def _same_key(a, b) -> bool:
    """Equality of two DeviceCsr._tensor_key() values: same tensor objects, same versions."""
    return (all(x is y for x, y in zip(a[0], b[0])) and a[1] == b[1] and a[2:] == b[2:])


def _offsets_tensor(ts, device):
    torch = _torch()
    if isinstance(ts, DeviceCsr):
        return ts.row_offsets, ts.rows, ts.nnz
    dev = _require_cuda(device)
    off = torch.as_tensor(np.ascontiguousarray(ts.offsets if hasattr(ts, "offsets") else
                                               [ts.atom_offset(t) for t in range(ts.num_tiles + 1)],
                                               dtype=np.int64)).to(dev)
    return off, ts.num_tiles, ts.num_atoms


def device_merge_path_partition(ts, lanes: int, device=None):
    """lw_merge_path_partition: torch int64 [(lanes+1), 2], bit-exact with the host."""
    torch = _torch()
    dev = ts.device if isinstance(ts, DeviceCsr) else (
        device if not isinstance(device, DeviceCsr) else device.device)
    off, rows, nnz = _offsets_tensor(ts, dev)
    out = torch.empty((lanes + 1, 2), dtype=torch.int64, device=off.device)
    bits = 32 if off.dtype == torch.int32 else 64
    lib = _lib.load()
    _lib.check(lib.lw_merge_path_partition(rows, nnz, off.data_ptr(), bits, lanes, out.data_ptr(),
                                           current_stream(off.device)), "lw_merge_path_partition")
    return out


def device_group_plan_prefix(ts, tiles_per_block: int, device=None):
    """lw_group_plan_prefix: torch int64 [nblocks, tpb+1]."""
    torch = _torch()
    off, rows, _ = _offsets_tensor(ts, device)
    nblocks = (rows + tiles_per_block - 1) // tiles_per_block
    out = torch.empty((nblocks, tiles_per_block + 1), dtype=torch.int64, device=off.device)
    bits = 32 if off.dtype == torch.int32 else 64
    lib = _lib.load()
    _lib.check(lib.lw_group_plan_prefix(rows, off.data_ptr(), bits, tiles_per_block, out.data_ptr(),
                                        current_stream(off.device)), "lw_group_plan_prefix")
    return out


def _csr_from_sorted_keys(n: int, scale: int, keys, seed: int, dtype, device) -> DeviceCsr:
    torch = _torch()
    rows = keys >> scale
    cols = (keys & (n - 1)).to(torch.int32)
    counts = torch.bincount(rows, minlength=n)
    nnz = int(keys.shape[0])
    odt = torch.int32 if nnz < (1 << 31) else torch.int64
    off = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(counts, 0, out=off[1:])
    vals = torch.empty(nnz, dtype=_torch_dtype(dtype), device=device)
    lib = _lib.load()
    _lib.check(lib.lw_hash_values(keys.data_ptr(), nnz, seed, _dtype_code(dtype), vals.data_ptr(),
                                  current_stream(device)), "lw_hash_values")
    return DeviceCsr(n, n, off.to(odt), cols, vals)


def generate_rmat_csr(scale: int, edge_factor: int = 16, seed: int = 3, a: float = 0.57,
                      b: float = 0.19, c: float = 0.19, dtype="float32", device=None,
                      chunk_edges: int = 1 << 27) -> DeviceCsr:
    """Directed R-MAT CSR built on the device: 2^scale rows, edge_factor*2^scale
    edges, duplicates removed, self-loops kept, no permutation; values are
    hash_values(key, seed) in U[-1, 1). Identical to the C oracle's lwo_rmat_csr.
    """
    from .sparse import rmat_thresholds

    torch = _torch()
    dev = _require_cuda(device)
    n = 1 << scale
    n_edges = edge_factor * n
    ta, tab, tabc = rmat_thresholds(a, b, c)
    lib = _lib.load()
    stream = current_stream(dev)
    uniq = []
    # generate + sort + dedup in chunks to bound the sort's scratch memory
    for start in range(0, n_edges, chunk_edges):
        cnt = min(chunk_edges, n_edges - start)
        k = torch.empty(cnt, dtype=torch.int64, device=dev)
        _lib.check(lib.lw_rmat_keys(scale, start, cnt, ta, tab, tabc, seed, k.data_ptr(), stream),
                   "lw_rmat_keys")
        uniq.append(torch.unique(k))
        del k
    keys = torch.unique(torch.cat(uniq)) if len(uniq) > 1 else uniq[0]
    del uniq
    return _csr_from_sorted_keys(n, scale, keys, seed, dtype, dev)


def generate_uniform_device(rows: int, cols: int, nnz_target: int, seed: int, dtype="float32",
                            device=None, chunk: int = 1 << 27) -> DeviceCsr:
    """Uniform-random rows x cols CSR built on the device (the C2u / C4-uniform
    inputs): nnz_target positions drawn uniformly from [0, rows*cols) with
    lw_uniform_key, duplicates removed (so nnz <= nnz_target, short by about
    nnz^2 / (2 rows cols)), values hash_values(row*cols + col, seed) in U[-1, 1).
    The reference's own generate_random_csr (sparse.py:164-187) draws exactly
    nnz_target distinct positions with NumPy and takes minutes at 32M atoms; the
    oracle's lwo_uniform_keys evaluates the same key function on the host."""
    torch = _torch()
    dev = _require_cuda(device)
    if rows < 1 or cols < 1 or nnz_target < 0:
        raise ValueError("rows, cols must be positive and nnz_target non-negative")
    space = rows * cols
    lib = _lib.load()
    stream = current_stream(dev)
    uniq = []
    for start in range(0, nnz_target, chunk):
        cnt = min(chunk, nnz_target - start)
        k = torch.empty(cnt, dtype=torch.int64, device=dev)
        _lib.check(lib.lw_uniform_keys(space, start, cnt, seed, k.data_ptr(), stream), "lw_uniform_keys")
        uniq.append(torch.unique(k))
        del k
    if not uniq:
        keys = torch.empty(0, dtype=torch.int64, device=dev)
    else:
        keys = torch.unique(torch.cat(uniq)) if len(uniq) > 1 else uniq[0]
    del uniq
    r = keys // cols
    counts = torch.bincount(r, minlength=rows)
    nnz = int(keys.shape[0])
    off = torch.zeros(rows + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=off[1:])
    vals = torch.empty(nnz, dtype=_torch_dtype(dtype), device=dev)
    if nnz:
        _lib.check(lib.lw_hash_values(keys.data_ptr(), nnz, seed, _dtype_code(dtype), vals.data_ptr(),
                                      stream), "lw_hash_values")
    odt = torch.int32 if nnz < (1 << 31) else torch.int64
    return DeviceCsr(rows, cols, off.to(odt), (keys - r * cols).to(torch.int32), vals)


def generate_banded_device(rows: int, half_bandwidth: int, seed: int, dtype="float32",
                           device=None) -> DeviceCsr:
    """Banded matrix (sparse.generate_banded_csr) built directly on the device."""
    torch = _torch()
    dev = _require_cuda(device)
    i = torch.arange(rows, dtype=torch.int64, device=dev)
    lo = torch.clamp(i - half_bandwidth, min=0)
    hi = torch.clamp(i + half_bandwidth + 1, max=rows)
    lengths = hi - lo
    off = torch.zeros(rows + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lengths, 0, out=off[1:])
    nnz = int(off[-1].item())
    owner = torch.repeat_interleave(i, lengths)
    cols = torch.arange(nnz, dtype=torch.int64, device=dev) - off[:-1][owner] + lo[owner]
    keys = owner * rows + cols
    vals = torch.empty(nnz, dtype=_torch_dtype(dtype), device=dev)
    lib = _lib.load()
    _lib.check(lib.lw_hash_values(keys.data_ptr(), nnz, seed, _dtype_code(dtype), vals.data_ptr(),
                                  current_stream(dev)), "lw_hash_values")
    odt = torch.int32 if nnz < (1 << 31) else torch.int64
    return DeviceCsr(rows, rows, off.to(odt), cols.to(torch.int32), vals)
