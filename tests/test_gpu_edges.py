"""GPU edge cases across the kernels: degenerate shapes, strided / misaligned
operands, zero-weight and self-loop graphs, 64-bit offsets — each checked
against the C oracle (bit-exact where the data are integers)."""

import numpy as np
import pytest

from conftest import integer_csr
from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2301_04792_b200 as lwb  # noqa: E402
from paper_2301_04792_b200 import DeviceCsr, ExecutorConfig, ScheduleKind  # noqa: E402

KINDS = list(ScheduleKind)


def dev(m, dtype="float64", offset_bits=None):
    return DeviceCsr.from_host(m, dtype=dtype, offset_bits=offset_bits)


def test_spmm_degenerate_shapes():
    m = lwb.generate_random_csr(30, 20, 100, seed=1)
    A = dev(m)
    for kind in KINDS:
        cfg = ExecutorConfig(schedule=kind)
        C = lwb.spmm(A, torch.ones(20, 0, dtype=torch.float64, device="cuda"), cfg)
        assert C.shape == (30, 0)
        empty = dev(lwb.CsrMatrix(0, 20, np.zeros(1, np.int64), [], []))
        assert lwb.spmm(empty, torch.ones(20, 3, dtype=torch.float64, device="cuda"), cfg).shape == (0, 3)
        nonz = dev(lwb.CsrMatrix(5, 20, np.zeros(6, np.int64), [], []))
        C = lwb.spmm(nonz, torch.ones(20, 3, dtype=torch.float64, device="cuda"), cfg)
        assert torch.equal(C, torch.zeros(5, 3, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("kind", KINDS)
def test_strided_and_misaligned_operands(kind):
    """x as a strided view; B as a transposed view and as an 8-byte-offset slice
    (the scalar path of the 16-byte-vector kernels)."""
    rng = np.random.default_rng(4)
    m = integer_csr(rng, 150, 120, 1500)
    A = dev(m, "float32")
    cfg = ExecutorConfig(schedule=kind)
    xs = torch.as_tensor(rng.integers(-3, 4, size=240).astype(np.float32), device="cuda")[::2]
    want = oracle.spmv(m.row_offsets, m.col_indices, m.values, xs.double().cpu().numpy(), "thread-mapped", lanes=1)
    np.testing.assert_array_equal(lwb.spmv(A, xs, cfg).double().cpu().numpy(), want)
    Bt = torch.as_tensor(rng.integers(-3, 4, size=(8, 120)).astype(np.float32), device="cuda").t()
    Bm = torch.as_tensor(rng.integers(-3, 4, size=(120 * 8 + 2,)).astype(np.float32), device="cuda")[2:].view(120, 8)
    for B in (Bt, Bm):
        want = oracle.spmm(m.row_offsets, m.col_indices, m.values, B.double().cpu().numpy(), "thread-mapped", lanes=1)
        np.testing.assert_array_equal(lwb.spmm(A, B, cfg).double().cpu().numpy(), want)


@pytest.mark.parametrize("bits", [32, 64])
def test_traversal_zero_weights_self_loops(bits):
    """Zero-weight edges, self-loops and duplicate distances: dist equal to the
    oracle (and to Dijkstra) bit for bit; BFS from an isolated vertex."""
    rng = np.random.default_rng(8)
    n = 400
    m = lwb.generate_random_csr(n, n, 3000, seed=3)
    w = rng.integers(0, 3, size=m.nnz).astype(np.float64)   # many zero weights
    off = m.row_offsets
    col = m.col_indices.copy()
    col[::17] = np.repeat(np.arange(n), np.diff(off))[::17]      # self-loops
    csr = lwb.coo_to_csr(lwb.CooMatrix(n, n, np.repeat(np.arange(n), np.diff(off)), col, w))
    G = dev(csr, offset_bits=bits)
    for kind in KINDS:
        cfg = ExecutorConfig(schedule=kind)
        src = int(np.argmax(np.diff(csr.row_offsets)))
        np.testing.assert_array_equal(lwb.sssp(G, src, cfg).cpu().numpy(),
                                      oracle.sssp(csr.row_offsets, csr.col_indices, csr.values, src))
        np.testing.assert_array_equal(lwb.bfs(G, src, cfg).cpu().numpy(),
                                      oracle.bfs(csr.row_offsets, csr.col_indices, src))
    iso = lwb.Graph(lwb.CsrMatrix(3, 3, [0, 0, 1, 1], [0], [1.0]))
    np.testing.assert_array_equal(lwb.bfs(iso, 0), [0, -1, -1])
    np.testing.assert_array_equal(lwb.sssp(iso, 0), [0.0, np.inf, np.inf])


def test_mmio_special_values_roundtrip_to_device():
    """Values Python's float() accepts (exponents, inf) survive parse -> CSR -> GPU."""
    text = ("%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 1e-300\n2 2 -2.5E+10\n"
            "3 1 inf\n3 3 +0.125\n")
    coo = lwb.parse_matrix_market(text)
    np.testing.assert_array_equal(coo.data, [1e-300, -2.5e10, np.inf, 0.125])
    csr = lwb.coo_to_csr(coo)
    y = lwb.spmv(csr, np.array([1.0, 1.0, 0.0]))
    assert y[0] == 1e-300 and y[1] == -2.5e10 and np.isinf(y[2])


def test_concurrent_streams_use_separate_workspaces():
    """work_oriented SpMV on two streams at once (each stream gets its own
    workspace): both results match the single-stream ones."""
    rng = np.random.default_rng(12)
    mats = [integer_csr(rng, 20_000, 20_000, 400_000), integer_csr(rng, 30_000, 25_000, 300_000)]
    A = [dev(m, "float32") for m in mats]
    xs = [torch.as_tensor(rng.integers(-2, 3, size=a.cols).astype(np.float32), device="cuda") for a in A]
    cfg = ExecutorConfig(schedule=ScheduleKind.MERGE_PATH)
    want = [lwb.spmv(a, x, cfg) for a, x in zip(A, xs)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [[], []]
    for _ in range(20):
        for k in range(2):
            with torch.cuda.stream(streams[k]):
                outs[k].append(lwb.spmv(A[k], xs[k], cfg))
    torch.cuda.synchronize()
    for k in range(2):
        for y in outs[k]:
            assert torch.equal(y, want[k])


def test_out_buffers_are_validated():
    """out= must be a contiguous buffer of the right shape, dtype and device."""
    m = lwb.generate_random_csr(50, 40, 300, seed=2)
    A = dev(m, "float32")
    x = torch.ones(40, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        lwb.spmv(A, x, out=torch.empty(100, dtype=torch.float32, device="cuda")[::2])
    with pytest.raises(ValueError):
        lwb.spmv(A, x, out=torch.empty(50, dtype=torch.float64, device="cuda"))
    B = torch.ones(40, 3, dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        lwb.spmm(A, B, out=torch.empty(3, 50, dtype=torch.float32, device="cuda").t())
    y = lwb.spmv(A, x, out=torch.empty(50, dtype=torch.float32, device="cuda"))
    np.testing.assert_allclose(y.cpu().numpy(), lwb.spmv(m, np.ones(40)), rtol=1e-5, atol=1e-5)
