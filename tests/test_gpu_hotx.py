"""GPU tests of the hot-x column packing (csrc/hotx.cu).

The packing is a B200 layout step in front of the work_oriented SpMV, not a
reference function, so its contract is checked two ways:
  * the inspector: hot set, slot order and relabeled col_indices equal a NumPy
    restatement of the rule (H = {c : count(c) >= T}, T the smallest threshold
    >= 2 with |H| <= max_hot; slots in ascending column order);
  * the executor: y from the packed kernel is bit-identical to the unpacked
    work_oriented kernel, and within the north-star tolerance of the C oracle.
"""

import functools

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2301_04792_b200 as lwb  # noqa: E402
from paper_2301_04792_b200 import DeviceCsr, ExecutorConfig, ScheduleKind  # noqa: E402

WO = ExecutorConfig(schedule=ScheduleKind.MERGE_PATH)
RTOL = {torch.float32: 1e-5, torch.float64: 1e-12}


def expected_hot(col, cols, max_hot):
    counts = np.bincount(np.asarray(col, np.int64), minlength=cols)
    if max_hot <= 0:
        return np.zeros(0, np.int64)
    vals = np.sort(counts)[::-1]
    # smallest T >= 2 with |{count >= T}| <= max_hot
    thr = max(2, int(vals[max_hot]) + 1) if max_hot < cols else 2
    return np.flatnonzero(counts >= thr)


def dev(off, col, val, cols, dtype, bits=32):
    odt = torch.int32 if bits == 32 else torch.int64
    return DeviceCsr(len(off) - 1, int(cols), torch.as_tensor(np.asarray(off, np.int64)).to("cuda", odt),
                     torch.as_tensor(np.asarray(col, np.int64)).to("cuda", torch.int32),
                     torch.as_tensor(np.asarray(val, np.float64)).to("cuda", dtype))


@functools.lru_cache(maxsize=None)
def skewed_csr(rows, cols, per_row, seed, hot_cols=0, hot_every=1):
    """Rows with Zipf-like column choices; optionally `hot_cols` columns in every
    hot_every-th row (counts above 2^16 push the radix select into its second pass)."""
    rng = np.random.default_rng(seed)
    off, col = [0], []
    for r in range(rows):
        k = int(rng.integers(0, 2 * per_row + 1))
        c = set((rng.zipf(1.3, k) - 1) % cols)
        if hot_cols and r % hot_every == 0:
            c |= set(range(hot_cols))
        c = sorted(c)
        col.extend(c)
        off.append(len(col))
    val = rng.uniform(-1, 1, len(col))
    return np.asarray(off), np.asarray(col, np.int64), val


CASES = [
    ("zipf", dict(rows=3000, cols=5000, per_row=12, seed=1), 256),
    ("zipf_small_cap", dict(rows=3000, cols=5000, per_row=12, seed=2), 7),
    ("all_fit", dict(rows=500, cols=300, per_row=8, seed=3), 32768),
    ("none", dict(rows=500, cols=300, per_row=8, seed=4), 0),
    ("two_pass", dict(rows=70000, cols=40000, per_row=2, seed=5, hot_cols=3), 1000),
    ("two_pass_tight", dict(rows=140000, cols=40000, per_row=1, seed=6, hot_cols=40, hot_every=2), 20),
]


@pytest.mark.parametrize("name,spec,max_hot", CASES, ids=[c[0] for c in CASES])
def test_inspector_matches_rule(name, spec, max_hot):
    off, col, val = skewed_csr(**spec)
    cols = spec["cols"]
    m = dev(off, col, val, cols, torch.float32)
    hx = m.pack_hot_columns(max_hot)
    want = expected_hot(col, cols, max_hot)
    assert hx.n_hot == len(want) <= max_hot
    assert np.array_equal(hx.hot_cols.cpu().numpy(), want)
    slot = np.full(cols, -1, np.int64)
    slot[want] = np.arange(len(want))
    exp = np.where(slot[col] >= 0, slot[col] | (1 << 31), col).astype(np.uint32).view(np.int32)
    assert np.array_equal(hx.packed.col_indices.cpu().numpy(), exp)
    assert torch.equal(hx.original_col_indices(), m.col_indices)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("bits", [32, 64])
@pytest.mark.parametrize("name,spec,max_hot", CASES, ids=[c[0] for c in CASES])
def test_packed_spmv_bit_identical(name, spec, max_hot, dtype, bits):
    off, col, val = skewed_csr(**spec)
    cols = spec["cols"]
    m = dev(off, col, val, cols, dtype, bits)
    x = np.random.default_rng(42).random(cols)
    xt = torch.as_tensor(x).to("cuda", dtype)
    y_plain = lwb.spmv(m, xt, WO)
    m.pack_hot_columns(max_hot)
    y_hot = lwb.spmv(m, xt, WO)
    assert torch.equal(y_hot, y_plain)
    for lanes in (1, 3, 97):
        cfg = ExecutorConfig(schedule=ScheduleKind.MERGE_PATH, lanes=lanes)
        m.drop_hot_columns()
        a = lwb.spmv(m, xt, cfg)
        m.pack_hot_columns(max_hot)
        assert torch.equal(lwb.spmv(m, xt, cfg), a)
    y_ref = oracle.spmv(off, col, val, x, "thread-mapped", lanes=1)
    ok, worst = oracle.tolerance_ok(y_hot.double().cpu().numpy(), y_ref,
                                    oracle.abs_row_sums(off, col, val, x), RTOL[dtype])
    assert ok, worst


def test_packing_follows_tensor_identity_and_other_schedules():
    off, col, val = skewed_csr(rows=800, cols=900, per_row=6, seed=9)
    m = dev(off, col, val, 900, torch.float32)
    hx = m.pack_hot_columns(64)
    assert m.hot_columns() is hx and m.pack_hot_columns(64) is hx
    x = torch.rand(900, device="cuda")
    # other schedules ignore the packing and run on the original col_indices
    for kind in (ScheduleKind.THREAD_MAPPED, ScheduleKind.GROUP_MAPPED):
        y = lwb.spmv(m, x, ExecutorConfig(schedule=kind))
        m.drop_hot_columns()
        assert torch.equal(y, lwb.spmv(m, x, ExecutorConfig(schedule=kind)))
        m.pack_hot_columns(64)
    # probes run the unpacked instrumented kernel and still attribute every atom once
    y, probe, _ = lwb.spmv_probe(m, x, WO)
    assert (probe["atom_visits"] == 1).all()
    # replacing a tensor invalidates the packing
    m.col_indices = m.col_indices.clone()
    assert m.hot_columns() is None


def test_empty_and_degenerate():
    m = dev([0, 0, 0], [], [], 5, torch.float32)
    hx = m.pack_hot_columns()
    assert hx.n_hot == 0
    assert torch.equal(lwb.spmv(m, torch.rand(5, device="cuda"), WO), torch.zeros(2, device="cuda"))
    m = dev([0], [], [], 0, torch.float32)
    m.pack_hot_columns()
    assert lwb.spmv(m, torch.zeros(0, device="cuda"), WO).numel() == 0
    # one column gathered by every row: the single hot slot
    rows = 1000
    m = dev(np.arange(rows + 1), np.zeros(rows, np.int64), np.ones(rows), 4, torch.float32)
    hx = m.pack_hot_columns(1)
    assert hx.n_hot == 1 and int(hx.hot_cols[0]) == 0
    x = torch.tensor([2.0, 0, 0, 0], device="cuda")
    assert torch.equal(lwb.spmv(m, x, WO), torch.full((rows,), 2.0, device="cuda"))


def test_rejects_bad_arguments():
    off, col, val = skewed_csr(rows=100, cols=100, per_row=4, seed=11)
    m = dev(off, col, val, 100, torch.float32)
    with pytest.raises(Exception):
        m.pack_hot_columns(32769)
    with pytest.raises(Exception):
        m.pack_hot_columns(-1)


def test_rmat_packed_bit_identical():
    m = lwb.generate_rmat_csr(16, 16, seed=3)
    x = torch.rand(m.cols, device="cuda")
    y = lwb.spmv(m, x, WO)
    hx = m.pack_hot_columns()
    assert 0 < hx.n_hot <= 12288
    assert torch.equal(lwb.spmv(m, x, WO), y)


def test_power_iteration_packed_iterates_bit_identical():
    """C5's driver over a packed operand: the iterates and norms equal the unpacked run."""
    from paper_2301_04792_b200.distributed import RowShard, nnz_balanced_bounds, power_iteration

    A = lwb.generate_rmat_csr(16, 8, seed=11)
    shard = RowShard(nnz_balanced_bounds(A.row_offsets.cpu().numpy(), 1), 0)
    x1, n1 = power_iteration(lambda x: lwb.spmv(A, x, WO), A.rows, shard, 6, dtype=torch.float32,
                             device="cuda")
    A.pack_hot_columns()
    x2, n2 = power_iteration(lambda x: lwb.spmv(A, x, WO), A.rows, shard, 6, dtype=torch.float32,
                             device="cuda")
    assert torch.equal(x1, x2) and n1 == n2


def test_fused_power_iteration_packed_bit_identical():
    """The SpMV-with-peer-writes kernel over a packed operand (world 1: the rank's own
    next-x buffer is its only peer) gives the unpacked iterates exactly."""
    from paper_2301_04792_b200.distributed import (RowShard, nnz_balanced_bounds,
                                                   power_iteration_fused)

    A = lwb.generate_rmat_csr(16, 8, seed=12)
    shard = RowShard(nnz_balanced_bounds(A.row_offsets.cpu().numpy(), 1), 0)
    x1, n1 = power_iteration_fused(A, A.rows, shard, 6)
    A.pack_hot_columns()
    x2, n2 = power_iteration_fused(A, A.rows, shard, 6)
    torch.cuda.synchronize()
    assert torch.equal(x1, x2) and n1 == n2


def test_peers_hotx_kernel_writes_every_buffer_at_the_row_base():
    """lw_spmv_work_oriented_peers_hotx: the packed peers kernel writes y and every peer
    buffer at row_base with the unpacked kernel's rows, bit for bit."""
    import ctypes

    from paper_2301_04792_b200 import _lib

    A = lwb.generate_rmat_csr(15, 8, seed=4)
    x = torch.rand(A.cols, device="cuda")
    want = lwb.spmv(A, x, WO)
    hx = A.pack_hot_columns()
    bufs = [torch.full((A.rows + 50,), -7.0, device="cuda") for _ in range(2)]
    y = torch.empty(A.rows, device="cuda")
    lib = _lib.load()
    need = lib.lw_spmv_work_oriented_hotx_workspace(A.rows, A.nnz, 0, hx.n_hot, _lib.LW_F32)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    ptrs = (ctypes.c_uint64 * 2)(*[b.data_ptr() for b in bufs])
    rc = lib.lw_spmv_work_oriented_peers_hotx(hx.packed.c_struct(), hx.hot_cols.data_ptr(), hx.n_hot,
                                              x.data_ptr(), y.data_ptr(), 0, ws.data_ptr(), need, 2,
                                              ptrs, 0, 25, torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.equal(y, want)
    for b in bufs:
        assert torch.equal(b[25:25 + A.rows], want)
        assert (b[:25] == -7.0).all() and (b[25 + A.rows:] == -7.0).all()
