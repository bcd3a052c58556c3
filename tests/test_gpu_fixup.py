"""The work_oriented carry fix-up (reference kernels.py:90-91: carries added to
their rows in lane order) as a segmented reduction: rows whose carries span
many lanes, runs that cross the fix-up kernel's CTAs (1024 carries each), one
row spanning every lane of a 2^28-atom matrix, and its cost."""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2301_04792_b200 as lwb  # noqa: E402
from paper_2301_04792_b200 import DeviceCsr, ExecutorConfig, ScheduleKind, _lib  # noqa: E402
from paper_2301_04792_b200.device import current_stream  # noqa: E402

WO = ScheduleKind.WORK_ORIENTED


def _dev(off, col, val, cols, dtype):
    return DeviceCsr(len(off) - 1, cols, torch.as_tensor(off).cuda().to(torch.int32),
                     torch.as_tensor(col).cuda().to(torch.int32), torch.as_tensor(val).cuda().to(dtype))


@pytest.mark.parametrize("lanes", [1500, 9000, 100_000, 1_500_000])
def test_runs_crossing_fixup_ctas_integer_bit_exact(lanes):
    """Rows of 2..20000 atoms cut into many lanes: runs of carries of every
    length, many crossing the 1024-carry CTAs of the fix-up. Integer data: the
    result must equal the reference merge-path fp64 sums bit for bit."""
    rng = np.random.default_rng(5)
    lengths = rng.integers(0, 20000, size=400)
    lengths[rng.random(400) < 0.3] = 0
    off = np.zeros(401, np.int64)
    np.cumsum(lengths, out=off[1:])
    nnz = int(off[-1])
    col = rng.integers(0, 5000, size=nnz)
    val = rng.integers(-3, 4, size=nnz).astype(np.float64)
    x = rng.integers(-3, 4, size=5000).astype(np.float64)
    want = oracle.spmv(off, col, val, x, "merge-path", lanes=lanes, threads=oracle.default_threads())
    m = _dev(off, col, val, 5000, torch.float64)
    y = lwb.spmv(m, torch.as_tensor(x).cuda(), ExecutorConfig(schedule=WO, lanes=lanes))
    np.testing.assert_array_equal(y.cpu().numpy(), want)


def _giant(dtype, nnz=1 << 28, cols=1 << 20):
    """3 short rows, then one row of `nnz` atoms (it spans every lane of the
    auto-sized launch), then empty rows and 2 short rows."""
    pre = 3 * 7
    off = np.array([0, 7, 14, 21, 21 + nnz, 21 + nnz, 21 + nnz, 28 + nnz, 35 + nnz], np.int64)
    total = int(off[-1])
    col = torch.arange(total, device="cuda", dtype=torch.int64) % cols
    g = torch.Generator(device="cuda").manual_seed(3)
    if dtype == torch.float64:   # integer data: sums exact in fp64
        val = torch.randint(-3, 4, (total,), device="cuda", generator=g).to(dtype)
        x = torch.randint(-3, 4, (cols,), device="cuda", generator=g).to(dtype)
    else:
        val = torch.rand(total, device="cuda", generator=g, dtype=dtype) * 2 - 1
        x = torch.rand(cols, device="cuda", generator=g, dtype=dtype)
    m = DeviceCsr(len(off) - 1, cols, torch.as_tensor(off).cuda().to(torch.int32),
                  col.to(torch.int32), val)
    assert pre == 21
    return m, x


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_one_row_spanning_every_lane(dtype):
    m, x = _giant(dtype)
    cfg = lwb.device_config(ExecutorConfig(schedule=WO), m)
    assert cfg.lanes > 60_000   # ~66 K lanes, every one of them carries into the giant row
    y = lwb.spmv(m, x, ExecutorConfig(schedule=WO)).cpu().numpy()
    host = [t.cpu().numpy() for t in (m.row_offsets, m.col_indices, m.values)]
    y_ref, scale = oracle.spmv_narrow(*host, x.cpu().numpy())
    if dtype == torch.float64:
        np.testing.assert_array_equal(y, y_ref)
    else:
        worst, row = oracle.worst_ratio(y, y_ref, scale, 1e-5)
        assert worst <= 1.0, (row, worst)


def test_one_row_spanning_several_merge_passes():
    """2.1 M lanes: the fix-up's last CTA merges > 4 K edge pieces in several
    1024-slot passes, all of one run carried from pass to pass (integer data,
    bit-exact)."""
    m, x = _giant(torch.float64)
    y = lwb.spmv(m, x, ExecutorConfig(schedule=WO, lanes=2_100_000)).cpu().numpy()
    host = [t.cpu().numpy() for t in (m.row_offsets, m.col_indices, m.values)]
    y_ref, _ = oracle.spmv_narrow(*host, x.cpu().numpy())
    np.testing.assert_array_equal(y, y_ref)


def test_fixup_cost_bounded_on_the_spanning_row():
    """The fix-up phase alone (lw_spmv_work_oriented_phases mask 4) on ~66 K
    carries that all belong to one row: one scan step per CTA, no serial walk."""
    m, x = _giant(torch.float32)
    lib = _lib.load()
    A = m.c_struct()
    y = torch.empty(m.rows, dtype=m.dtype, device="cuda")
    need = lib.lw_spmv_work_oriented_workspace(m.rows, m.nnz, 0, A.dtype)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    s = current_stream(m.device)

    def phase(mask):
        _lib.check(lib.lw_spmv_work_oriented_phases(A, x.data_ptr(), y.data_ptr(), 0, ws.data_ptr(),
                                                    need, mask, s), "phases")

    phase(1)
    phase(2)
    for _ in range(3):
        phase(4)
    ts = []
    for _ in range(20):
        phase(1)   # the partition phase re-arms the fix-up ticket
        phase(2)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        phase(4)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = float(np.median(ts))
    print(f"fix-up over the spanning row: {us:.1f} us")
    assert us <= 20.0, f"fix-up took {us:.1f} us"
