"""GPU parity for SpMM (C = A B) under the three schedules, through the C ABI.

Follows the reference's SpMM tests (tests/test_kernels.py:70-102, SPEC.md:399,
431-432): golden outputs recorded from lanework.spmm, integer data bit-exact
across every schedule, lane count and dtype, column slices equal to SpMV, a
single column degenerating to SpMV, and the north star's tolerance
|C - C_ref| <= rtol * sum_j |A_ij B_jc| (rtol 1e-5 fp32, 1e-12 fp64) otherwise.
"""

import numpy as np
import pytest

from conftest import integer_csr, unpack
from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2301_04792_b200 as lwb  # noqa: E402
from paper_2301_04792_b200 import DeviceCsr, ExecutorConfig, ScheduleKind  # noqa: E402

RTOL = {torch.float32: 1e-5, torch.float64: 1e-12}
KINDS = {"thread-mapped": ScheduleKind.THREAD_MAPPED, "merge-path": ScheduleKind.MERGE_PATH,
         "group-mapped": ScheduleKind.GROUP_MAPPED}


def dev_csr(off, col, val, cols, dtype=torch.float64, offset_bits=32):
    odt = torch.int32 if offset_bits == 32 else torch.int64
    return DeviceCsr(len(off) - 1, int(cols), torch.as_tensor(np.asarray(off, np.int64)).to("cuda", odt),
                     torch.as_tensor(np.asarray(col, np.int64)).to("cuda", torch.int32),
                     torch.as_tensor(np.asarray(val, np.float64)).to("cuda", dtype))


def run(m, B, kind, lanes=None, gs=32, tpb=None):
    cfg = ExecutorConfig(schedule=KINDS[kind], lanes=lanes, group_size=gs, tiles_per_block=tpb)
    Bt = torch.as_tensor(np.asarray(B, np.float64)).to("cuda", m.dtype)
    return lwb.spmm(m, Bt, cfg).double().cpu().numpy()


def test_spmm_matches_reference_golden(golden):
    g = golden["spmm"]
    cases = list(golden.spmm_cases())
    for ck, (mi, ci, integer) in enumerate(g["meta"]):
        _, off, col, val, B, rows, cols = cases[mi]
        m = dev_csr(off, col, val, cols)
        kind = str(g["cfg_kind"][ci])
        C = run(m, B, kind, lanes=int(g["cfg_lanes"][ci]), gs=int(g["cfg_gs"][ci]),
                tpb=int(g["cfg_tpb"][ci]))
        want = unpack(g["C"], g["C_idx"], ck).reshape(rows, B.shape[1])
        if integer or kind == "group-mapped":
            # group_mapped sums each C[tile, :] in the reference's member-major
            # order with unfused fp64 ops (k_spmm_group_tiles): bit-identical
            np.testing.assert_array_equal(C, want, err_msg=f"case {ck} {kind}")
        else:
            ok, worst = oracle.tolerance_ok(C, want, oracle.abs_spmm_sums(off, col, val, B), 1e-12)
            assert ok, f"case {ck} {kind}: worst {worst:.3g}"


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8, 16, 24, 64, 130, 257])
def test_integer_spmm_bit_identical_across_schedules(dtype, n):
    """Acceptance criterion 4 for SpMM: every schedule, lane
    count and group shape gives the same bits on integer data (vector and scalar
    paths, one slab and several)."""
    rng = np.random.default_rng(n)
    m = integer_csr(rng, 300, 200, 3000)
    B = rng.integers(-3, 4, size=(200, n)).astype(np.float64)
    want = oracle.spmm(m.row_offsets, m.col_indices, m.values, B, "thread-mapped", lanes=1)
    dm = dev_csr(m.row_offsets, m.col_indices, m.values, m.cols, dtype)
    for kind, lanes, gs in [("thread-mapped", None, 32), ("thread-mapped", 7, 32),
                            ("merge-path", None, 32), ("merge-path", 1, 32), ("merge-path", 13, 32),
                            ("merge-path", 3300, 32), ("group-mapped", None, 32),
                            ("group-mapped", 40, 4), ("group-mapped", None, 256)]:
        C = run(dm, B, kind, lanes=lanes, gs=gs)
        np.testing.assert_array_equal(C, want, err_msg=f"{kind} lanes={lanes} gs={gs} n={n}")


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_spmm_tolerance_power_law(dtype):
    m = lwb.generate_power_law_csr(5000, 12.0, 1.2, seed=9)
    B = np.random.default_rng(42).random((m.cols, 16)) - 0.5
    ref = oracle.spmm(m.row_offsets, m.col_indices, m.values, B, "thread-mapped", lanes=1)
    scale = oracle.abs_spmm_sums(m.row_offsets, m.col_indices, m.values, B)
    dm = dev_csr(m.row_offsets, m.col_indices, m.values, m.cols, dtype)
    for kind in KINDS:
        C = run(dm, B, kind)
        ok, worst = oracle.tolerance_ok(C, ref, scale, RTOL[dtype])
        assert ok, f"{kind}: worst {worst:.3g}"


def test_spmm_column_slices_equal_spmv():
    """column c of spmm(m, B) equals spmv(m, B[:, c]) exactly on integer data."""
    rng = np.random.default_rng(3)
    m = integer_csr(rng, 120, 90, 1500)
    B = rng.integers(-3, 4, size=(90, 5)).astype(np.float64)
    dm = dev_csr(m.row_offsets, m.col_indices, m.values, m.cols, torch.float32)
    for kind in KINDS:
        C = run(dm, B, kind)
        for c in range(5):
            x = torch.as_tensor(B[:, c]).to("cuda", torch.float32)
            y = lwb.spmv(dm, x, ExecutorConfig(schedule=KINDS[kind])).double().cpu().numpy()
            np.testing.assert_array_equal(C[:, c], y)


def test_spmm_host_api_and_errors():
    """Reference signature/behaviour: host operands give an fp64 NumPy C; a B with
    the wrong shape raises ValueError (kernels.py:133-134); an empty matrix gives 0."""
    m = lwb.CsrMatrix(2, 2, [0, 2, 3], [0, 1, 1], [1.0, 2.0, 3.0])
    C = lwb.spmm(m, np.array([[1.0, 2.0], [3.0, 4.0]]))
    assert C.dtype == np.float64
    np.testing.assert_array_equal(C, [[7.0, 10.0], [9.0, 12.0]])
    with pytest.raises(ValueError):
        lwb.spmm(m, np.ones((3, 2)))
    with pytest.raises(ValueError):
        lwb.spmm(m, np.ones(2))
    empty = lwb.CsrMatrix(4, 4, np.zeros(5, np.int64), [], [])
    for kind in KINDS.values():
        np.testing.assert_array_equal(lwb.spmm(empty, np.ones((4, 3)), ExecutorConfig(schedule=kind)),
                                      np.zeros((4, 3)))


@pytest.mark.parametrize("bits", [32, 64])
def test_spmm_long_row_split_across_lanes(bits):
    """One 200k-atom row cut across many merge-path lanes: carries fixed up in order."""
    nnz = 200_000
    off = np.array([0, 3, nnz - 5, nnz - 5, nnz])
    rng = np.random.default_rng(1)
    col = rng.integers(0, 64, size=nnz)
    val = rng.integers(-2, 3, size=nnz).astype(np.float64)
    B = rng.integers(-2, 3, size=(64, 8)).astype(np.float64)
    dm = dev_csr(off, col, val, 64, torch.float64, offset_bits=bits)
    want = oracle.spmm(off, col, val, B, "thread-mapped", lanes=1)
    for lanes in (None, 5, 999):
        np.testing.assert_array_equal(run(dm, B, "merge-path", lanes=lanes), want)
