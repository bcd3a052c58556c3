"""N>1 path on CPU: nnz-balanced row shards and the power-iteration all-gather,
run with world_size 2 over gloo. The per-shard SpMV is the C oracle here (the
checker); on GPUs the same driver calls the CUDA kernels and NCCL."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2301_04792_b200 as lw
from paper_2301_04792_b200.distributed import (RowShard, nnz_balanced_bounds, power_iteration,
                                               shard_of)


def test_bounds_properties():
    m = lw.generate_power_law_csr(5000, 16.0, 1.1, seed=3)
    off = m.row_offsets
    for parts in (1, 2, 3, 4, 8, 64):
        b = nnz_balanced_bounds(off, parts)
        assert b[0] == 0 and b[-1] == m.rows and np.all(np.diff(b) >= 0)
        shard_nnz = np.diff(off[b])
        # each shard is within one row of the ideal share
        ideal = m.nnz / parts
        max_row = int(np.diff(off).max())
        assert np.all(shard_nnz <= ideal + max_row + 1)
    b = nnz_balanced_bounds(np.array([0, 0, 0]), 4)
    assert b[0] == 0 and b[-1] == 2
    with pytest.raises(ValueError):
        nnz_balanced_bounds(off, 0)


def test_shards_reassemble_the_product():
    from oracle import oracle

    m = lw.generate_power_law_csr(3000, 12.0, 1.3, seed=5)
    x = np.random.default_rng(1).random(m.cols)
    want = oracle.spmv(m.row_offsets, m.col_indices, m.values, x, "merge-path", lanes=64)
    b = nnz_balanced_bounds(m.row_offsets, 4)
    parts = []
    for r in range(4):
        s = shard_of(m, b, r)
        parts.append(oracle.spmv(s.row_offsets, s.col_indices, s.values, x, "merge-path", lanes=16))
    np.testing.assert_allclose(np.concatenate(parts), want, rtol=1e-12, atol=1e-12)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out, chunks=1):
    from oracle import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = lw.generate_power_law_csr(4000, 10.0, 1.2, seed=7)
        b = nnz_balanced_bounds(m.row_offsets, world)
        shard = RowShard(b, rank)
        mine = shard_of(m, b, rank)

        def local(x, r0=0, r1=None):
            part = shard_of(mine, [0, r0, mine.rows if r1 is None else r1], 1)
            y = oracle.spmv(part.row_offsets, part.col_indices, part.values,
                            x.double().numpy(), "merge-path", lanes=32)
            return torch.from_numpy(y).to(x.dtype)

        x, norms = power_iteration(local, m.rows, shard, iters=8, dtype=torch.float64,
                                   chunks=chunks)
        out[rank] = (x.numpy().copy(), list(norms))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunks", [1, 3])
def test_power_iteration_world2_matches_single_process(chunks):
    """chunks=3: the overlapped path (per-chunk async all-gathers + reorder)."""
    from oracle import oracle

    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, port, out, chunks), nprocs=2, join=True,
                       start_method="spawn")
    m = lw.generate_power_law_csr(4000, 10.0, 1.2, seed=7)
    x = np.full(m.rows, 1.0 / np.sqrt(m.rows))
    norms = []
    for _ in range(8):
        y = oracle.spmv(m.row_offsets, m.col_indices, m.values, x, "merge-path", lanes=32)
        n = np.linalg.norm(y)
        norms.append(n)
        x = y / n
    for r in range(2):
        xr, nr = out[r]
        np.testing.assert_allclose(xr, x, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(nr, norms, rtol=1e-12)
    np.testing.assert_array_equal(out[0][0], out[1][0])  # ranks stay identical


def test_chunked_single_process_equals_plain():
    """world 1: the chunked driver computes the same iterates as the plain one."""
    from oracle import oracle

    m = lw.generate_power_law_csr(2000, 8.0, 1.3, seed=11)
    b = nnz_balanced_bounds(m.row_offsets, 1)
    shard = RowShard(b, 0)

    def local(x, r0=0, r1=None):
        part = shard_of(m, [0, r0, m.rows if r1 is None else r1], 1)
        y = oracle.spmv(part.row_offsets, part.col_indices, part.values, x.double().numpy(),
                        "merge-path", lanes=16)
        return torch.from_numpy(y)

    x1, n1 = power_iteration(local, m.rows, shard, iters=5, dtype=torch.float64)
    x4, n4 = power_iteration(local, m.rows, shard, iters=5, dtype=torch.float64, chunks=4)
    # the per-chunk SpMV cuts rows differently (merge-path lanes), so only FP order differs
    np.testing.assert_allclose(x4.numpy(), x1.numpy(), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(n4, n1, rtol=1e-12)


def _worker_inplace(rank, world, port, out, chunks, exact=False):
    """The in-place gather layout: operator columns renamed into the gather
    buffer, SpMV writing its slot, all-gather in place, norm + scale in place."""
    from oracle import oracle
    from paper_2301_04792_b200.distributed import GatherLayout, power_iteration_inplace

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = lw.generate_power_law_csr(4000, 10.0, 1.2, seed=7)
        b = nnz_balanced_bounds(m.row_offsets, world)
        lay = GatherLayout(b, chunks, exact=exact)
        mine = lay.remap_columns(shard_of(m, b, rank))

        def local(x, r0, r1, out_view):
            part = shard_of(mine, [0, r0, r1], 1)
            out_view.copy_(torch.from_numpy(oracle.spmv(part.row_offsets, part.col_indices, part.values,
                                                        x.double().numpy(), "merge-path", lanes=32)))

        xb, norms = power_iteration_inplace(local, lay, 8, rank=rank, dtype=torch.float64)
        out[rank] = (lay.from_layout(xb).numpy().copy(), list(norms))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,chunks,exact", [(2, 1, False), (2, 3, False), (3, 2, False), (2, 1, True),
                                                (3, 2, True)])
def test_inplace_gather_layout_matches_single_process(world, chunks, exact):
    """Padded slots (equal-size NCCL all-gather) and the exact layout (uneven
    per-rank pieces; gloo emulates NCCL's uneven all_gather through a padded
    staging buffer) give the single-process iterates."""
    from oracle import oracle

    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker_inplace, args=(world, port, out, chunks, exact), nprocs=world, join=True,
                       start_method="spawn")
    m = lw.generate_power_law_csr(4000, 10.0, 1.2, seed=7)
    x = np.full(m.rows, 1.0 / np.sqrt(m.rows))
    norms = []
    for _ in range(8):
        y = oracle.spmv(m.row_offsets, m.col_indices, m.values, x, "merge-path", lanes=32)
        norms.append(np.linalg.norm(y))
        x = y / norms[-1]
    for r in range(world):
        xr, nr = out[r]
        np.testing.assert_allclose(xr, x, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(nr, norms, rtol=1e-12)
    np.testing.assert_array_equal(out[0][0], out[world - 1][0])


def test_gather_layout_positions():
    from paper_2301_04792_b200.distributed import GatherLayout

    b = np.array([0, 5, 12, 13])
    lay = GatherLayout(b, chunks=2)
    # slots: chunk 0 widths max(2, 3, 0)=3, chunk 1 max(3, 4, 1)=4 -> size 3*3 + 3*4
    assert lay.widths == [3, 4] and lay.size == 21
    assert sorted(lay.pos.tolist()) == sorted(set(lay.pos.tolist()))   # injective
    v = torch.arange(13, dtype=torch.float64)
    np.testing.assert_array_equal(lay.from_layout(lay.to_layout(v)).numpy(), v.numpy())
    buf = lay.to_layout(v)
    pad = np.setdiff1d(np.arange(lay.size), lay.pos)
    assert (buf[torch.as_tensor(pad)] == 0).all()


def test_exact_gather_layout_is_the_vector():
    from paper_2301_04792_b200.distributed import GatherLayout

    b = np.array([0, 5, 12, 13])
    lay = GatherLayout(b, chunks=2, exact=True)
    assert lay.size == 13 and (lay.pos == np.arange(13)).all()
    assert lay.pieces(0) == [(0, 2), (5, 3), (12, 0)] and lay.pieces(1) == [(2, 3), (8, 4), (12, 1)]
    assert lay.slot(1, 1) == (8, 4, 3, 7)
    m = lw.generate_power_law_csr(50, 4.0, 1.5, seed=1)
    assert lay.remap_columns(m) is m


def test_work_balanced_bounds_are_merge_path_tiles():
    """The rows+nnz split is the tile column of the reference merge-path partition
    (schedules.py:88-110), rows whole, and balances rows + nnz within one row."""
    from paper_2301_04792_b200.distributed import row_bounds, work_balanced_bounds
    from paper_2301_04792_b200.schedules import merge_path_partition
    from paper_2301_04792_b200.work import TileSet

    rng = np.random.default_rng(7)
    lengths = rng.integers(0, 40, size=5000)
    lengths[rng.random(5000) < 0.4] = 0
    off = np.concatenate([[0], np.cumsum(lengths)])
    for parts in (1, 2, 3, 4, 8, 13):
        b = work_balanced_bounds(off, parts)
        assert b[0] == 0 and b[-1] == off.size - 1 and (np.diff(b) >= 0).all()
        np.testing.assert_array_equal(b[1:-1], merge_path_partition(TileSet(off), parts)[1:-1, 0])
        items = (off[b[1:]] + b[1:]) - (off[b[:-1]] + b[:-1])
        assert items.max() - items.min() <= 2 * (lengths.max() + 1) + 2
        np.testing.assert_array_equal(row_bounds(off, parts, "work"), b)
        np.testing.assert_array_equal(row_bounds(off, parts, "nnz"), nnz_balanced_bounds(off, parts))
        c = row_bounds(off, parts)   # default: nnz + ROW_COST * rows
        cost = off + 1.75 * np.arange(off.size)
        per = cost[c[1:]] - cost[c[:-1]]
        assert c[0] == 0 and c[-1] == off.size - 1 and (np.diff(c) >= 0).all()
        assert per.max() - per.min() <= 2 * (lengths.max() + 1.75) + 1e-9
    with pytest.raises(ValueError):
        row_bounds(off, 2, "rows")
