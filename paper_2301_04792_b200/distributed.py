"""Multi-GPU SpMV: nnz-balanced row shards, x replicated, NCCL all-gather of y.

Rows (tiles) are independent, so one SpMV needs no exchange when
every rank holds all of x: rank k computes y[r_k:r_{k+1}] from its row shard.
Only the iterated SpMV (power iteration, BASELINE config C5) has a real
exchange step — y becomes the next x on every rank — and that is one
all-gather(v) of the uneven y shards per iteration over NVLink/NVSwitch.

The per-shard SpMV is a parameter (``local_spmv``) so the same driver runs the
CUDA kernels in production and a CPU checker under gloo in the tests.
"""

from __future__ import annotations

import numpy as np

__all__ = ["nnz_balanced_bounds", "work_balanced_bounds", "weighted_bounds", "row_bounds", "shard_of", "power_iteration", "power_iteration_fused",
           "power_iteration_graph", "power_iteration_inplace", "chunk_bounds", "RowShard",
           "GatherLayout"]


def nnz_balanced_bounds(row_offsets, parts: int) -> np.ndarray:
    """Row boundaries r_0=0 <= r_1 <= ... <= r_G=rows with ~nnz/G atoms per shard.

    r_k = (first row whose prefix reaches k*nnz/G): searchsorted(off, k*nnz/G,
    'left') over the row offsets, so each shard is within one row of perfect
    nnz balance. Deterministic integer arithmetic, identical on every rank.
    """
    off = np.asarray(row_offsets, dtype=np.int64)
    if parts < 1:
        raise ValueError("parts must be >= 1")
    rows, nnz = off.size - 1, int(off[-1])
    targets = (np.arange(parts + 1, dtype=np.int64) * nnz) // parts
    b = np.searchsorted(off, targets, side="left").astype(np.int64)
    b = np.minimum(b, rows)
    b[0], b[-1] = 0, rows
    return np.maximum.accumulate(b)


def work_balanced_bounds(row_offsets, parts: int) -> np.ndarray:
    """Row boundaries that balance rows + nnz (merge-path items) instead of nnz:
    the tile coordinates of merge_path_partition(ts, parts) (reference
    schedules.py:88-110), i.e. the work_oriented schedule applied across GPUs.
    A shard's SpMV costs about one item per row plus one per atom, so a shard of
    many short or empty rows (R-MAT's high row ids; the tail of a degree-sorted
    operator) is no longer the slowest one. Rows stay whole."""
    from .schedules import merge_path_partition
    from .work import TileSet

    off = np.asarray(row_offsets, dtype=np.int64)
    if parts < 1:
        raise ValueError("parts must be >= 1")
    b = merge_path_partition(TileSet(off), parts)[:, 0].astype(np.int64)
    b[0], b[-1] = 0, off.size - 1
    return np.maximum.accumulate(b)


def weighted_bounds(row_offsets, parts: int, row_weight: float) -> np.ndarray:
    """Row boundaries balancing nnz + row_weight * rows (whole rows): b_k is the
    first row whose prefix cost off[t] + w*t reaches k/parts of the total. A
    vectorised bisection over the parts+1 targets (no rows-sized temporaries:
    C5's 67 M offsets would need two 0.5 GB cost arrays per rank)."""
    off = np.asarray(row_offsets, dtype=np.int64)
    if parts < 1:
        raise ValueError("parts must be >= 1")
    if row_weight < 0:
        raise ValueError("row_weight must be >= 0")
    rows = off.size - 1
    w = float(row_weight)
    total = float(off[-1]) + w * rows
    targets = total * np.arange(parts + 1, dtype=np.float64) / parts
    lo = np.zeros(parts + 1, dtype=np.int64)           # first t with cost(t) >= target
    hi = np.full(parts + 1, rows, dtype=np.int64)
    while (lo < hi).any():
        mid = (lo + hi) // 2
        ge = off[mid].astype(np.float64) + w * mid >= targets
        hi = np.where(ge, mid, hi)
        lo = np.where(ge, lo, mid + 1)
    b = lo
    b[0], b[-1] = 0, rows
    return np.maximum.accumulate(b)


# Measured cost of one row relative to one atom in a shard's work_oriented SpMV
# step (least squares over per-shard times of C3 at 1-8 shards, B200: 3.4 us per
# M atoms, 5.9 us per M rows; tools/shard_projection.py).
ROW_COST = 1.75


def row_bounds(row_offsets, parts: int, balance: str = "cost") -> np.ndarray:
    """Shard boundaries by ``balance``: "cost" (nnz + ROW_COST * rows, the
    measured per-shard cost; default), "work" (rows + nnz, the merge-path tiles,
    work_balanced_bounds), "nnz" (nnz_balanced_bounds, the north star's split) or
    "w<float>" (nnz + w * rows)."""
    if balance == "cost":
        return weighted_bounds(row_offsets, parts, ROW_COST)
    if balance == "work":
        return work_balanced_bounds(row_offsets, parts)
    if balance == "nnz":
        return nnz_balanced_bounds(row_offsets, parts)
    if balance.startswith("w"):
        try:
            w = float(balance[1:])
        except ValueError:
            w = None
        if w is not None and w >= 0:
            return weighted_bounds(row_offsets, parts, w)
    raise ValueError(f"unknown balance {balance!r}")


class RowShard:
    """Rank-local view: rows [r0, r1) of the global matrix."""

    def __init__(self, bounds, rank: int):
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.rank = rank
        self.r0, self.r1 = int(self.bounds[rank]), int(self.bounds[rank + 1])

    @property
    def rows(self) -> int:
        return self.r1 - self.r0

    @property
    def counts(self) -> list[int]:
        return [int(v) for v in np.diff(self.bounds)]


def shard_of(host_csr, bounds, rank: int):
    """Host CSR of rows [bounds[rank], bounds[rank+1]) with rebased offsets."""
    from .sparse import CsrMatrix

    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    off = host_csr.row_offsets[r0:r1 + 1]
    a0, a1 = int(off[0]), int(off[-1])
    return CsrMatrix(r1 - r0, host_csr.cols, off - a0, host_csr.col_indices[a0:a1],
                     host_csr.values[a0:a1])


def chunk_bounds(rows: int, chunks: int) -> np.ndarray:
    """Split local rows [0, rows) into ``chunks`` contiguous, near-equal pieces."""
    chunks = max(1, int(chunks))
    return (np.arange(chunks + 1, dtype=np.int64) * rows) // chunks


class _Completed:
    """A finished exchange (the synchronous gloo emulation) with the async API."""

    def wait(self):
        return None


_DONE = _Completed()
_UNEVEN_OK = [True]   # cleared if the NCCL backend rejects an uneven all_gather


class GatherLayout:
    """Where each row of the full vector sits in the all-gather buffer.

    The shards' row counts are uneven (nnz-balanced bounds), NCCL's all-gather
    moves equal slots, so slot (chunk k, rank r) holds width_k = max_r(rows of
    chunk k of rank r) entries: the buffer is chunk-major, rank-major, with
    zero padding after each slot's real rows. ``pos[i]`` is the buffer index of
    global row i. Renaming the operator's columns through ``pos`` once
    (``remap_columns``) lets every iteration read x straight out of the
    gathered buffer: the SpMV writes its rows into its own slot, NCCL gathers
    in place, the norm and the scaling run over the buffer (padding stays 0) —
    no send copy, concatenation or reorder pass per iteration."""

    def __init__(self, bounds, chunks: int = 1, exact: bool = False):
        b = np.asarray(bounds, dtype=np.int64)
        self.world = b.size - 1
        self.chunks = max(1, int(chunks))
        self.bounds = b
        counts = np.diff(b)
        self.cb = [chunk_bounds(int(c), self.chunks) for c in counts]
        # exact: no padding — the buffer is the vector itself (pos = identity) and
        # chunk k is exchanged as uneven per-rank pieces (NCCL's all_gather with
        # uneven outputs: one broadcast per rank, grouped), so a shard with many
        # more rows than the others (R-MAT's sparse tail; the degree-sorted C5
        # operator puts 86% of the rows on the last of 8 shards) costs no padding
        self.exact = bool(exact)
        if self.exact:
            self.widths = [0] * self.chunks
            self.offs = np.zeros(self.chunks + 1, dtype=np.int64)
            self.size = int(b[-1])
            self.pos = np.arange(self.size, dtype=np.int64)
            self._pos_dev = {}
            return
        self.widths = [max(int(self.cb[r][k + 1] - self.cb[r][k]) for r in range(self.world))
                       for k in range(self.chunks)]
        self.offs = np.concatenate([[0], np.cumsum([self.world * w for w in self.widths])]).astype(np.int64)
        self.size = int(self.offs[-1])
        pos = np.empty(int(b[-1]), dtype=np.int64)
        for r in range(self.world):
            for k in range(self.chunks):
                lo, hi = int(b[r] + self.cb[r][k]), int(b[r] + self.cb[r][k + 1])
                base = int(self.offs[k] + r * self.widths[k])
                pos[lo:hi] = base + np.arange(hi - lo)
        self.pos = pos
        self._pos_dev = {}

    def pos_on(self, device):
        """``pos`` as an int64 tensor on ``device`` (uploaded once per device)."""
        import torch

        key = str(device)
        if key not in self._pos_dev:
            self._pos_dev[key] = torch.as_tensor(self.pos, device=device)
        return self._pos_dev[key]

    def slot(self, rank: int, k: int) -> tuple[int, int, int, int]:
        """(buffer start of my slot, slot width, local row range r0, r1) of chunk k."""
        r0, r1 = int(self.cb[rank][k]), int(self.cb[rank][k + 1])
        if self.exact:
            return int(self.bounds[rank]) + r0, r1 - r0, r0, r1
        return int(self.offs[k] + rank * self.widths[k]), self.widths[k], r0, r1

    def pieces(self, k: int) -> list[tuple[int, int]]:
        """exact layout: (start, length) of chunk k of every rank in the vector."""
        return [(int(self.bounds[r] + self.cb[r][k]), int(self.cb[r][k + 1] - self.cb[r][k]))
                for r in range(self.world)]

    def exchange(self, buf, k: int, rank: int, group=None):
        """Async all-gather of chunk k into ``buf`` in place; returns the work."""
        import torch
        import torch.distributed as dist

        if not self.exact:
            lo, hi = int(self.offs[k]), int(self.offs[k + 1])
            start = int(self.offs[k] + rank * self.widths[k])
            return dist.all_gather_into_tensor(buf[lo:hi], buf[start:start + self.widths[k]], group=group,
                                               async_op=True)
        views = [buf[a:a + n] for a, n in self.pieces(k)]
        if dist.get_backend(group) == "nccl" and _UNEVEN_OK[0]:   # grouped broadcasts, exact bytes
            try:
                return dist.all_gather(views, views[rank], group=group, async_op=True)
            except (RuntimeError, ValueError):   # a build without uneven all_gather: pad instead
                _UNEVEN_OK[0] = False
        # (gloo only gathers equal sizes: pad through a staging buffer)
        w = max(n for _, n in self.pieces(k)) if self.world else 0
        tmp = torch.zeros(self.world * w, dtype=buf.dtype, device=buf.device)
        mine = torch.zeros(w, dtype=buf.dtype, device=buf.device)
        mine[: views[rank].numel()].copy_(views[rank])
        dist.all_gather_into_tensor(tmp, mine, group=group)
        for r, v in enumerate(views):
            v.copy_(tmp[r * w: r * w + v.numel()])
        return _DONE

    def remap_columns(self, m):
        """The operator with column c renamed pos[c] (host CsrMatrix or DeviceCsr);
        its column count becomes the buffer size."""
        from .sparse import CsrMatrix

        if self.exact:   # pos is the identity
            return m
        if isinstance(m, CsrMatrix):
            return CsrMatrix(m.rows, self.size, m.row_offsets, self.pos[m.col_indices], m.values)
        import torch

        from .device import DeviceCsr

        pos = torch.as_tensor(self.pos.astype(np.int32), device=m.device)
        col = pos.index_select(0, m.col_indices.to(torch.int64)) if m.nnz else m.col_indices.clone()
        return DeviceCsr(m.rows, self.size, m.row_offsets, col, m.values)

    def to_layout(self, x):
        """Full vector -> buffer form (zeros in the padding)."""
        import torch

        out = torch.zeros(self.size, dtype=x.dtype, device=x.device)
        out[self.pos_on(x.device)] = x
        return out

    def from_layout(self, buf):
        return buf.index_select(0, self.pos_on(buf.device))


def power_iteration_inplace(local_spmv, layout: GatherLayout, iters: int, rank: int = 0, group=None,
                            x0=None, dtype=None, device=None, _norms_out=None):
    """power_iteration over a GatherLayout: x lives in the gather buffer form.

    ``local_spmv(x_buf, r0, r1, out)`` writes this rank's local rows [r0, r1)
    (operator columns remapped with ``layout.remap_columns``) into ``out``, a
    view of this rank's slot. Per iteration and chunk k: the SpMV writes the
    slot, an async NCCL all-gather fills chunk k of the next buffer in place
    (overlapping chunk k+1's SpMV); then one norm read and one in-place scaling
    of the buffer. Two buffers alternate (x_k is read while x_{k+1} is
    gathered). Returns (x in buffer form, norms); ``layout.from_layout`` maps it
    back once."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world != layout.world:
        raise ValueError(f"layout built for {layout.world} ranks, group has {world}")
    dt = dtype or torch.float32
    bufs = [torch.zeros(layout.size, dtype=dt, device=device) for _ in range(2)]
    if x0 is None:
        n = layout.pos.size
        bufs[0].copy_(layout.to_layout(torch.full((n,), 1.0 / np.sqrt(n), dtype=dt, device=device)))
    else:
        bufs[0].copy_(x0)
    norms = []
    cur = 0
    for it in range(iters):
        x, nxt = bufs[cur], bufs[1 - cur]
        works = []
        for k in range(layout.chunks):
            start, width, r0, r1 = layout.slot(rank, k)
            local_spmv(x, r0, r1, nxt[start:start + (r1 - r0)])
            if world > 1:
                works.append(layout.exchange(nxt, k, rank, group))
        for w in works:
            w.wait()
        nrm = _normalise_into(nxt)
        if _norms_out is not None:
            _norms_out[it].copy_(nrm)
        else:
            norms.append(nrm)
        cur = 1 - cur
    if _norms_out is not None:
        return bufs[cur], None
    return bufs[cur], [float(v) for v in norms]


def _normalise_into(y):
    """||y||_2 (device fp64 scalar) and y /= ||y|| in place (library kernels on
    CUDA; torch on CPU for the gloo tests)."""
    import torch

    if not y.is_cuda:
        nrm = torch.linalg.vector_norm(y, dtype=torch.float64)
        if nrm > 0:
            y.copy_((y / nrm).to(y.dtype))
        return nrm
    from . import _lib
    from .device import _dtype_code, current_stream

    lib = _lib.load()
    code = _dtype_code(y.dtype)
    stream = current_stream(y.device)
    ws = _NORM_WS.get(max(lib.lw_norm_workspace(y.numel()), 8), y.device, stream)
    nrm = torch.empty((), dtype=torch.float64, device=y.device)
    _lib.check(lib.lw_vector_norm(y.data_ptr(), y.numel(), code, ws.data_ptr(), ws.numel(),
                                  nrm.data_ptr(), stream), "lw_vector_norm")
    _lib.check(lib.lw_vector_scale(y.data_ptr(), y.numel(), code, nrm.data_ptr(), y.data_ptr(),
                                   stream), "lw_vector_scale")
    return nrm


def power_iteration_graph(local_spmv, n: int, shard: RowShard, iters: int, group=None,
                          device=None, dtype=None):
    """power_iteration captured once into a CUDA graph and replayed.

    The ``iters`` iterations (SpMV launches, the NCCL all-gather when N > 1, the
    norm/scale kernels) are recorded into one torch.cuda.CUDAGraph on the first
    call after a warm-up run, so a replay costs one launch instead of ~6 per
    iteration; ``local_spmv`` must write into a fixed output buffer and allocate
    nothing on the library side (the package's kernels take cached workspaces).
    Returns a callable: ``run(x0=None) -> (x, norms)``.
    """
    import torch

    dt = dtype or torch.float32
    x_in = torch.full((n,), 1.0 / np.sqrt(n), dtype=dt, device=device)
    # warm-up outside capture: library attributes, workspaces, NCCL communicators
    power_iteration(local_spmv, n, shard, 1, group=group, x0=x_in.clone())
    torch.cuda.synchronize(device)
    norms_t = torch.empty(iters, dtype=torch.float64, device=device)
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream(device)
    side.wait_stream(torch.cuda.current_stream(device))
    with torch.cuda.stream(side):
        with torch.cuda.graph(g):
            x_out, _ = power_iteration(local_spmv, n, shard, iters, group=group, x0=x_in,
                                       on_iter=None, _norms_out=norms_t)
    torch.cuda.current_stream(device).wait_stream(side)

    def run(x0=None):
        x_in.copy_(x0 if x0 is not None else torch.full_like(x_in, 1.0 / np.sqrt(n)))
        g.replay()
        return x_out, [float(v) for v in norms_t.cpu()]

    run.graph = g
    return run


def power_iteration(local_spmv, n: int, shard: RowShard, iters: int, group=None, x0=None,
                    device=None, dtype=None, on_iter=None, chunks: int = 1, _norms_out=None):
    """x_{k+1} = A x_k / ||A x_k||_2 for ``iters`` iterations, y all-gathered.

    ``local_spmv(x_full) -> y_shard`` computes this rank's rows; with
    ``chunks > 1`` it is called as ``local_spmv(x_full, r0, r1)`` for local row
    ranges and must return those rows.

    Over NCCL with uneven shards the exchange is exact: each rank's rows (per
    chunk) go out as one piece of an uneven all_gather straight into the full y
    (grouped broadcasts, no padding). Otherwise (gloo, even shards):
    chunks == 1: the uneven shards are padded to the largest shard so one
    all_gather_into_tensor moves them.
    chunks > 1: the shard is cut into row chunks (every rank uses the same count,
    so chunk k of every rank is exchanged together); chunk k's all-gather is
    issued asynchronously as soon as its SpMV is enqueued, so it runs on NCCL's
    stream while chunk k+1's SpMV computes (at 8 GPUs the exchange
    is as long as the SpMV, so it has to overlap). One index_select then puts the
    rank-major, chunk-major pieces back in row order.

    Every rank normalises the same full y locally (identical arithmetic on every
    rank, no all-reduce). Returns (x, norms) with norms[k] = ||A x_k||.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    counts = shard.counts
    width = max(counts) if counts else 0
    if x0 is None:
        x = torch.full((n,), 1.0 / np.sqrt(n), dtype=dtype or torch.float32, device=device)
    else:
        x = x0
    chunks = max(1, int(chunks))
    even = all(c == width for c in counts)
    if world > 1 and chunks == 1:
        gathered = torch.empty(world * width, dtype=x.dtype, device=x.device)
        send = torch.zeros(width, dtype=x.dtype, device=x.device)
    if chunks > 1:
        # per-rank chunk sizes (every rank derives all of them from the bounds)
        cb = [chunk_bounds(c, chunks) for c in counts]
        widths = [max(int(cb[r][k + 1] - cb[r][k]) for r in range(len(counts))) for k in range(chunks)]
        mine = cb[shard.rank] if world > 1 else chunk_bounds(shard.rows, chunks)
        if world > 1:
            sends = [torch.zeros(w, dtype=x.dtype, device=x.device) for w in widths]
            recvs = [torch.empty(world * w, dtype=x.dtype, device=x.device) for w in widths]
            # row order: rank r, chunk k, element j  <-  recvs[k][r * widths[k] + j]
            offs = np.concatenate([[0], np.cumsum([world * w for w in widths])])
            idx = np.concatenate([offs[k] + r * widths[k] + np.arange(cb[r][k + 1] - cb[r][k])
                                  for r in range(world) for k in range(chunks)]).astype(np.int64)
            order = torch.as_tensor(idx, device=x.device)
    # NCCL gathers uneven pieces exactly (grouped broadcasts): no padding, y
    # assembled in row order in place (GatherLayout's exact mode, without the layout)
    exact = world > 1 and dist.get_backend(group) == "nccl" and not even and _UNEVEN_OK[0]
    if exact:
        y_full = torch.empty(n, dtype=x.dtype, device=x.device)
        b = shard.bounds
        cbs = [chunk_bounds(int(c), chunks) for c in counts]
        views = [[y_full[int(b[r] + cbs[r][c]): int(b[r] + cbs[r][c + 1])] for r in range(world)]
                 for c in range(chunks)]
    norms = []
    for k in range(iters):
        if exact:
            works = []
            for c in range(chunks):
                mine_c = views[c][shard.rank]
                r0 = int(cbs[shard.rank][c])
                mine_c.copy_(local_spmv(x, r0, r0 + mine_c.numel()) if chunks > 1 else local_spmv(x))
                try:
                    works.append(dist.all_gather(views[c], mine_c, group=group, async_op=True))
                except (RuntimeError, ValueError):   # no uneven all_gather: equal-size pieces
                    _UNEVEN_OK[0] = False
                    w = max(v.numel() for v in views[c])
                    tmp = torch.zeros(world * w, dtype=x.dtype, device=x.device)
                    pad = torch.zeros(w, dtype=x.dtype, device=x.device)
                    pad[: mine_c.numel()].copy_(mine_c)
                    dist.all_gather_into_tensor(tmp, pad, group=group)
                    for r, v in enumerate(views[c]):
                        v.copy_(tmp[r * w: r * w + v.numel()])
            for w in works:
                w.wait()
            y = y_full
        elif chunks == 1:
            y_local = local_spmv(x)
            if world > 1:
                send[: shard.rows].copy_(y_local)
                dist.all_gather_into_tensor(gathered, send, group=group)
                y = gathered if even else torch.cat(
                    [gathered[r * width: r * width + counts[r]] for r in range(world)])
            else:
                y = y_local
        elif world > 1:
            works = []
            for c in range(chunks):
                r0, r1 = int(mine[c]), int(mine[c + 1])
                sends[c][: r1 - r0].copy_(local_spmv(x, r0, r1))
                works.append(dist.all_gather_into_tensor(recvs[c], sends[c], group=group,
                                                         async_op=True))
            for w in works:
                w.wait()
            y = torch.cat(recvs).index_select(0, order)
        else:
            y = torch.cat([local_spmv(x, int(mine[c]), int(mine[c + 1])) for c in range(chunks)])
        # ||y|| in fp64 and x = y / ||y|| on the device; no host sync inside the loop
        nrm, x = _normalise(y, x.dtype)
        if _norms_out is not None:   # graph capture: norms stay on the device
            _norms_out[k].copy_(nrm)
        else:
            norms.append(nrm)
        if on_iter is not None:
            on_iter(k, x)
    if _norms_out is not None:
        return x, None
    return x, [float(v) for v in norms]


def _normalise(y, dtype):
    """(||y||_2 as a device fp64 scalar, y / ||y||): the library's deterministic
    norm + scale kernels for CUDA tensors (one read for the norm, one read + write
    for the scaling), torch for CPU tensors (the gloo tests)."""
    import torch

    if not y.is_cuda:
        nrm = torch.linalg.vector_norm(y, dtype=torch.float64)
        return nrm, torch.where(nrm > 0, y / nrm, y).to(dtype)
    from . import _lib
    from .device import _dtype_code, current_stream

    lib = _lib.load()
    y = y.contiguous()
    code = _dtype_code(y.dtype)
    need = lib.lw_norm_workspace(y.numel())
    stream = current_stream(y.device)
    ws = _NORM_WS.get(max(need, 8), y.device, stream)
    nrm = torch.empty((), dtype=torch.float64, device=y.device)
    _lib.check(lib.lw_vector_norm(y.data_ptr(), y.numel(), code, ws.data_ptr(), ws.numel(),
                                  nrm.data_ptr(), stream), "lw_vector_norm")
    x = torch.empty_like(y, dtype=dtype)
    if x.dtype != y.dtype:
        return nrm, torch.where(nrm > 0, y / nrm, y).to(dtype)
    _lib.check(lib.lw_vector_scale(y.data_ptr(), y.numel(), code, nrm.data_ptr(), x.data_ptr(),
                                   stream), "lw_vector_scale")
    return nrm, x


class _LazyWs:
    def __init__(self):
        self._ws = None

    def get(self, nbytes, device, stream=0):
        if self._ws is None:
            from .device import Workspace

            self._ws = Workspace()
        return self._ws.get(nbytes, device, stream)


_NORM_WS = _LazyWs()


def _spmv_peers(A, x, y, peer_ptrs, mc_ptr: int, row_base: int, ws, stream: int) -> None:
    import ctypes

    from . import _lib

    lib = _lib.load()
    arr = (ctypes.c_uint64 * max(1, len(peer_ptrs)))(*[int(p) for p in peer_ptrs])
    hx = A.hot_columns()
    if hx is not None:   # hot-x packed operand: same rows, bit for bit
        rc = lib.lw_spmv_work_oriented_peers_hotx(
            hx.packed.c_struct(), hx.hot_cols.data_ptr() if hx.n_hot else None, hx.n_hot,
            x.data_ptr(), y.data_ptr(), 0, ws.data_ptr(), ws.numel(), len(peer_ptrs), arr,
            int(mc_ptr), row_base, stream)
    else:
        rc = lib.lw_spmv_work_oriented_peers(A.c_struct(), x.data_ptr(), y.data_ptr(), 0, ws.data_ptr(),
                                             ws.numel(), len(peer_ptrs), arr, int(mc_ptr), row_base, stream)
    _lib.check(rc, "lw_spmv_work_oriented_peers")


def power_iteration_fused(A, n: int, shard: RowShard, iters: int, group=None, x0=None,
                          multicast: bool = True):
    """Power iteration with the all-gather fused into the SpMV (SURVEY §8(e) stretch).

    ``A`` is this rank's row shard (DeviceCsr, rows [shard.r0, shard.r1)). The
    next x lives in two symmetric-memory buffers (torch.distributed
    _symmetric_memory: every rank's copy is mapped into every other rank's
    address space over NVLink); the work_oriented SpMV kernel writes each row it
    produces straight into all of them (lw_spmv_work_oriented_peers: one NVLS
    multimem.st per row when the NVSwitch multicast object exists, else one P2P
    store per peer), a device-side barrier on the buffer's signal pads orders
    the writes before anyone reads, and every rank normalises its own full copy.
    No NCCL call and no separate gather pass: the exchange rides on the SpMV's
    own row writes. Buffers alternate between iterations, so one barrier per
    iteration suffices (a rank rewrites a buffer only after every rank has
    passed the barrier that follows its last read).

    world == 1 runs the same kernel path with ordinary buffers (no peers).
    Returns (x, norms) like power_iteration.
    """
    import torch
    import torch.distributed as dist

    from .device import Workspace, current_stream

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dev, dtype = A.values.device, A.values.dtype
    if world > 1:
        import torch.distributed._symmetric_memory as symm_mem

        g = group or dist.group.WORLD
        me = dist.get_rank(g)
        bufs = [symm_mem.empty(n, dtype=dtype, device=dev) for _ in range(2)]
        hdls = [symm_mem.rendezvous(b, g) for b in bufs]
        # the rank's own rows are the kernel's y (its slice of its own buffer); the
        # peer stores go to the other ranks' buffers only
        peers = [[p for i, p in enumerate(h.buffer_ptrs) if i != me] for h in hdls]
        mcs = [int(getattr(h, "multicast_ptr", 0) or 0) if multicast else 0 for h in hdls]
    else:
        bufs = [torch.empty(n, dtype=dtype, device=dev) for _ in range(2)]
        hdls = [None, None]
        peers = [[], []]
        mcs = [0, 0]
    x = torch.full((n,), 1.0 / np.sqrt(n), dtype=dtype, device=dev) if x0 is None else x0
    from . import _lib
    from .kernels import spmv as _spmv
    from .executor import ExecutorConfig
    from .schedules import ScheduleKind
    wo = ExecutorConfig(schedule=ScheduleKind.MERGE_PATH)

    hx = A.hot_columns()
    need = (_lib.load().lw_spmv_work_oriented_hotx_workspace(A.rows, A.nnz, 0, hx.n_hot, A.c_struct().dtype)
            if hx is not None else
            _lib.load().lw_spmv_work_oriented_workspace(A.rows, A.nnz, 0, A.c_struct().dtype))
    ws = Workspace().get(need, dev)
    stream = current_stream(dev)
    norms = []
    for k in range(iters):
        b = k % 2
        y_own = bufs[b][shard.r0: shard.r1]
        if peers[b] or mcs[b]:
            _spmv_peers(A, x, y_own, peers[b], mcs[b], shard.r0, ws, stream)
        else:   # nobody to send to (world 1): the SpMV writes the next x directly
            _spmv(A, x, wo, out=y_own)
        if hdls[b] is not None:
            hdls[b].barrier(channel=0)
        nrm, x = _normalise(bufs[b], dtype)
        norms.append(nrm)
    return x, [float(v) for v in norms]
