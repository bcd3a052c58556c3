"""The host-operand SpMV's overlapped download (kernels._spmv_host_overlapped):
spmv(CsrMatrix, ndarray) on a large matrix runs the merge-path (or
thread_mapped) SpMV in equal-row blocks, lightest first, and downloads each
block's y while the later blocks compute. Checked against the C oracle (reference kernels.py:57-98): integer
data bit-exact, real data within the north star's fp64 bound; ragged inputs
(empty rows at the block bounds, one row holding most atoms) included."""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu


def _matrix(rng, rows, cols, lengths, integer):
    import paper_2301_04792_b200 as lw

    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    col = rng.integers(0, cols, size=int(off[-1])).astype(np.int64)
    for r in range(rows):   # sorted columns per row, like the reference's CSR
        col[off[r]:off[r + 1]].sort()
    val = (rng.integers(-3, 4, size=col.size).astype(np.float64) if integer
           else rng.random(col.size) * 2 - 1)
    return lw.CsrMatrix(rows, cols, off, col, val)


@pytest.fixture
def small_threshold(monkeypatch):
    from paper_2301_04792_b200 import kernels

    monkeypatch.setattr(kernels, "_OVERLAP_MIN_NNZ", 1)
    return kernels


@pytest.mark.parametrize("integer", [True, False])
@pytest.mark.parametrize("shape", ["uniform", "empty_runs", "one_giant_row"])
@pytest.mark.parametrize("blocks", [2, 4, 7])
def test_overlapped_host_spmv_matches_oracle(small_threshold, monkeypatch, shape, integer, blocks):
    import paper_2301_04792_b200 as lw

    monkeypatch.setattr(small_threshold, "_OVERLAP_BLOCKS", blocks)
    rng = np.random.default_rng(blocks * 10 + len(shape))
    rows, cols = 20_000, 30_000
    if shape == "uniform":
        lengths = rng.integers(0, 30, size=rows)
    elif shape == "empty_runs":
        lengths = rng.integers(0, 30, size=rows)
        lengths[rows // 4: rows // 2] = 0
        lengths[-1000:] = 0
    else:
        lengths = rng.integers(0, 3, size=rows)
        lengths[rows // 3] = 400_000
    m = _matrix(rng, rows, cols, lengths, integer)
    x = rng.integers(-3, 4, size=cols).astype(np.float64) if integer else rng.random(cols)
    y = lw.spmv(m, x)
    assert m.__dict__["_lw_device_cache"], "the device copy must be cached"
    dm = next(iter(m.__dict__["_lw_device_cache"].values()))[1]
    assert "_lw_row_blocks" in dm.__dict__, "the overlapped path must have run"
    assert isinstance(y, np.ndarray) and y.dtype == np.float64 and y.shape == (rows,)
    want = oracle.spmv(m.row_offsets, m.col_indices, m.values, x, "merge-path", threads=4)
    if integer:
        np.testing.assert_array_equal(y, want)
    else:
        ok, worst = oracle.tolerance_ok(y, want, oracle.abs_row_sums(m.row_offsets, m.col_indices,
                                                                     m.values, x), 1e-12)
        assert ok, worst
    # a second call reuses the cached blocks and gives the same y
    np.testing.assert_array_equal(lw.spmv(m, x), y)


def test_overlapped_blocks_follow_rebinding(small_threshold):
    """Rebinding the matrix's values re-uploads and rebuilds the row blocks."""
    import paper_2301_04792_b200 as lw

    rng = np.random.default_rng(5)
    m = _matrix(rng, 5000, 5000, rng.integers(0, 20, size=5000), True)
    x = rng.integers(-3, 4, size=5000).astype(np.float64)
    y1 = lw.spmv(m, x)
    m.values = m.values * 2
    y2 = lw.spmv(m, x)
    np.testing.assert_array_equal(y2, 2 * y1)


def test_overlapped_thread_mapped_is_bit_identical(small_threshold):
    """thread_mapped row blocks: every row is one thread's ordered chain, so y
    equals the single-launch y bit for bit (real-valued data)."""
    import torch

    import paper_2301_04792_b200 as lw

    rng = np.random.default_rng(8)
    m = _matrix(rng, 30_000, 20_000, rng.integers(0, 60, size=30_000), False)
    x = rng.random(20_000)
    cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.THREAD_MAPPED)
    y = lw.spmv(m, x, cfg)
    dm = next(iter(m.__dict__["_lw_device_cache"].values()))[1]
    assert "_lw_row_blocks" in dm.__dict__
    single = lw.spmv(dm, torch.as_tensor(x, device="cuda"), cfg).cpu().numpy()
    np.testing.assert_array_equal(y, single)
    want = oracle.spmv(m.row_offsets, m.col_indices, m.values, x, "thread-mapped", threads=4)
    ok, worst = oracle.tolerance_ok(y, want, oracle.abs_row_sums(m.row_offsets, m.col_indices,
                                                                 m.values, x), 1e-12)
    assert ok, worst


def test_explicit_lanes_and_fp32_keep_the_single_launch(small_threshold):
    """An explicit lane count (the reference's P) or a non-fp64 device copy runs
    one launch over the whole matrix, as before."""
    import paper_2301_04792_b200 as lw

    rng = np.random.default_rng(6)
    m = _matrix(rng, 4000, 4000, rng.integers(0, 20, size=4000), True)
    x = rng.integers(-3, 4, size=4000).astype(np.float64)
    y = lw.spmv(m, x, lw.ExecutorConfig(lanes=96))
    dm = next(iter(m.__dict__["_lw_device_cache"].values()))[1]
    assert "_lw_row_blocks" not in dm.__dict__
    want = oracle.spmv(m.row_offsets, m.col_indices, m.values, x, "merge-path", lanes=96)
    np.testing.assert_array_equal(y, want)
    y32 = lw.spmv(m, x, dtype="float32")
    np.testing.assert_array_equal(y32, want)
