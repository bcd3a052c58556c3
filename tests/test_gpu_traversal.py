"""GPU parity for SSSP / BFS (frontier relaxation under every schedule), through
the C ABI, against golden outputs recorded from lanework.sssp / bfs (which equal
dijkstra / serial_bfs) and the C oracle: distances and depths must be
bit-identical (the converged relaxation has a unique fixed point)."""

import numpy as np
import pytest

from conftest import unpack
from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2301_04792_b200 as lwb  # noqa: E402
from paper_2301_04792_b200 import ExecutorConfig, ScheduleKind  # noqa: E402

CFGS = [(ScheduleKind.THREAD_MAPPED, None, 32), (ScheduleKind.THREAD_MAPPED, 3, 32),
        (ScheduleKind.MERGE_PATH, None, 32), (ScheduleKind.MERGE_PATH, 1, 32),
        (ScheduleKind.MERGE_PATH, 7, 32), (ScheduleKind.GROUP_MAPPED, None, 32),
        (ScheduleKind.GROUP_MAPPED, 12, 4), (ScheduleKind.GROUP_MAPPED, None, 256)]


def graphs(golden):
    g = golden["traversal"]
    for k, src in enumerate(g["src"]):
        off, col = unpack(g["off"], g["off_idx"], k), unpack(g["col"], g["col_idx"], k)
        w = unpack(g["w"], g["col_idx"], k)
        yield (lwb.Graph(lwb.CsrMatrix(len(off) - 1, len(off) - 1, off, col, w)), int(src),
               unpack(g["dist"], g["v_idx"], k), unpack(g["depth"], g["v_idx"], k))


def test_sssp_bfs_match_reference_golden(golden):
    for G, src, dist, depth in graphs(golden):
        for kind, lanes, gs in CFGS:
            cfg = ExecutorConfig(schedule=kind, lanes=lanes, group_size=gs)
            np.testing.assert_array_equal(lwb.sssp(G, src, cfg), dist, err_msg=f"{kind} {lanes}")
            np.testing.assert_array_equal(lwb.bfs(G, src, cfg), depth, err_msg=f"{kind} {lanes}")


def test_sssp_pass_api_host_state(golden):
    """sssp_init + sssp_pass loop (the reference's caller-owned convergence loop)."""
    for G, src, dist, _ in list(graphs(golden))[:5]:
        state = lwb.sssp_init(G.num_vertices, src)
        passes = 0
        while state.in_frontier.any():
            n = lwb.sssp_pass(G, state, ExecutorConfig(schedule=ScheduleKind.MERGE_PATH))
            assert n == int(state.out_frontier.sum())
            state.in_frontier = state.out_frontier
            passes += 1
            assert passes <= G.num_vertices + 1
        np.testing.assert_array_equal(state.dist, dist)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_rmat_sssp_bfs_device_path(dtype):
    """A 2^16-vertex R-MAT graph (|weights|) resident on the device: every schedule
    gives the oracle's distances and depths; results stay torch tensors."""
    A = lwb.generate_rmat_csr(16, 8, seed=7, dtype=dtype)
    A = lwb.DeviceCsr(A.rows, A.cols, A.row_offsets, A.col_indices, A.values.abs())
    off = A.row_offsets.cpu().numpy().astype(np.int64)
    col = A.col_indices.cpu().numpy().astype(np.int64)
    w = A.values.double().cpu().numpy()
    src = int(np.argmax(np.diff(off)))
    want_d, want_h = oracle.sssp(off, col, w, src), oracle.bfs(off, col, src)
    for kind, lanes, gs in CFGS:
        cfg = ExecutorConfig(schedule=kind, lanes=lanes, group_size=gs)
        d, passes = lwb.sssp(A, src, cfg, return_passes=True)
        assert isinstance(d, torch.Tensor) and d.is_cuda and passes >= 1
        np.testing.assert_array_equal(d.cpu().numpy(), want_d)
        np.testing.assert_array_equal(lwb.bfs(A, src, cfg).cpu().numpy(), want_h)


def test_traversal_errors_and_edges():
    m = lwb.CsrMatrix(3, 3, [0, 1, 2, 2], [1, 2], [1.5, 2.0])
    G = lwb.Graph(m)
    with pytest.raises(ValueError):
        lwb.sssp(G, 3)
    with pytest.raises(ValueError):
        lwb.bfs(G, -1)
    np.testing.assert_array_equal(lwb.sssp(G, 0), [0.0, 1.5, 3.5])
    np.testing.assert_array_equal(lwb.sssp(G, 2), [np.inf, np.inf, 0.0])
    np.testing.assert_array_equal(lwb.bfs(G, 1), [lwb.UNREACHED, 0, 1])
    # single vertex, no edges
    one = lwb.Graph(lwb.CsrMatrix(1, 1, [0, 0], [], []))
    np.testing.assert_array_equal(lwb.sssp(one, 0), [0.0])
    np.testing.assert_array_equal(lwb.bfs(one, 0), [0])
