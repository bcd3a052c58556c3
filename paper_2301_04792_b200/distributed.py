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

__all__ = ["nnz_balanced_bounds", "shard_of", "power_iteration", "RowShard"]


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


def power_iteration(local_spmv, n: int, shard: RowShard, iters: int, group=None, x0=None,
                    device=None, dtype=None, on_iter=None):
    """x_{k+1} = A x_k / ||A x_k||_2 for ``iters`` iterations, y all-gathered.

    ``local_spmv(x_full) -> y_shard`` computes this rank's rows. The uneven
    shards are padded to the largest shard so a single all_gather_into_tensor
    (NCCL all-gather over NVLink) moves them; every rank then holds the full y,
    normalises it locally (identical arithmetic on every rank, no all-reduce)
    and uses it as the next x. Returns (x, norms) with norms[k] = ||A x_k||.
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
    even = all(c == width for c in counts)
    if world > 1:
        gathered = torch.empty(world * width, dtype=x.dtype, device=x.device)
        send = torch.zeros(width, dtype=x.dtype, device=x.device)
    norms = []
    for k in range(iters):
        y_local = local_spmv(x)
        if world > 1:
            send[: shard.rows].copy_(y_local)
            dist.all_gather_into_tensor(gathered, send, group=group)
            y = gathered if even else torch.cat(
                [gathered[r * width: r * width + counts[r]] for r in range(world)])
        else:
            y = y_local
        # ||y|| accumulated in fp64 on the device; no host sync inside the loop
        nrm = torch.linalg.vector_norm(y, dtype=torch.float64)
        norms.append(nrm)
        x = torch.where(nrm > 0, y / nrm, y).to(x.dtype)
        if on_iter is not None:
            on_iter(k, x)
    return x, [float(v) for v in norms]
