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


def _worker(rank, world, port, out):
    from oracle import oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = lw.generate_power_law_csr(4000, 10.0, 1.2, seed=7)
        b = nnz_balanced_bounds(m.row_offsets, world)
        shard = RowShard(b, rank)
        mine = shard_of(m, b, rank)

        def local(x):
            y = oracle.spmv(mine.row_offsets, mine.col_indices, mine.values,
                            x.double().numpy(), "merge-path", lanes=32)
            return torch.from_numpy(y).to(x.dtype)

        x, norms = power_iteration(local, m.rows, shard, iters=8, dtype=torch.float64)
        out[rank] = (x.numpy().copy(), list(norms))
    finally:
        dist.destroy_process_group()


def test_power_iteration_world2_matches_single_process():
    from oracle import oracle

    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
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
