"""Pin the C oracle to the reference: every golden vector recorded from lanework
itself (tests/golden/make_golden.py) must be reproduced exactly (CPU only)."""

import numpy as np
import pytest

from conftest import unpack
from oracle import oracle

KIND_NAMES = ["thread-mapped", "merge-path", "group-mapped"]


def test_oracle_builds_and_loads():
    assert oracle.lib().lwo_version() == 1


def test_merge_path_search_every_diagonal(golden):
    g = golden["schedules"]
    for s, off in enumerate(golden.tile_sets()):
        want = unpack(g["search"], g["search_idx"], s).reshape(-1, 2)
        got = np.array([oracle.merge_path_search(off, d) for d in range(want.shape[0])])
        np.testing.assert_array_equal(got.reshape(-1, 2), want)
        # and the brute-force walk (reference tests/conftest.py:40-54) agrees
        np.testing.assert_array_equal(np.array(oracle.merge_walk_coords(off)), want)


def test_merge_path_partition(golden):
    g = golden["schedules"]
    k = 0
    for off in golden.tile_sets():
        for p in g["lane_counts"]:
            want = unpack(g["parts"], g["parts_idx"], k).reshape(-1, 2)
            np.testing.assert_array_equal(oracle.merge_path_partition(off, int(p)), want)
            np.testing.assert_array_equal(oracle.merge_path_partition(off, int(p), threads=3), want)
            k += 1


def test_per_lane_counts_match_reference_imbalance(golden):
    g = golden["schedules"]
    shapes = g["gm_shapes"]
    k = 0
    for off in golden.tile_sets():
        for p in g["lane_counts"]:
            for kind in KIND_NAMES:
                for gs, tpb in (shapes if kind == "group-mapped" else [(32, 32)]):
                    want = unpack(g["imbal"], g["imbal_idx"], k)
                    la, _, _ = oracle.assignment(off, kind, int(p), int(gs), int(tpb))
                    np.testing.assert_array_equal(la, want, err_msg=f"{kind} P={p} gs={gs}")
                    k += 1


def test_assignment_maps_match_reference_executors(golden):
    g = golden["schedules"]
    sets = golden.tile_sets()
    for k, (si, p, ki, gs, tpb) in enumerate(g["assign_meta"]):
        _, al, at = oracle.assignment(sets[si], KIND_NAMES[ki], int(p), int(gs), int(tpb))
        np.testing.assert_array_equal(al, unpack(g["assign_lane"], g["assign_idx"], k))
        np.testing.assert_array_equal(at, unpack(g["assign_tile"], g["assign_idx"], k))


@pytest.mark.parametrize("threads", [1, 2, 3])
def test_spmv_matches_reference(golden, threads):
    g = golden["spmv"]
    cases = list(golden.spmv_cases())
    for yk, (mi, ci, integer) in enumerate(g["meta"]):
        _, off, col, val, x, rows, cols = cases[mi]
        y = oracle.spmv(off, col, val, x, str(g["cfg_kind"][ci]), lanes=int(g["cfg_lanes"][ci]),
                        threads=threads, group_size=int(g["cfg_gs"][ci]),
                        tiles_per_block=int(g["cfg_tpb"][ci]))
        want = unpack(g["y"], g["y_idx"], yk)
        if integer:
            np.testing.assert_array_equal(y, want)
        else:
            scale = oracle.abs_row_sums(off, col, val, x)
            assert oracle.tolerance_ok(y, want, scale, 1e-12)[0]


def test_spmv_known_answers():
    # reference tests/test_kernels.py:19-34
    y = oracle.spmv([0, 2, 3], [0, 1, 1], [1.0, 2.0, 3.0], np.ones(2), "merge-path", lanes=3)
    np.testing.assert_array_equal(y, [3.0, 3.0])
    for kind in KIND_NAMES:
        np.testing.assert_array_equal(oracle.spmv(np.zeros(5, np.int64), [], [], np.ones(4), kind,
                                                  lanes=4), np.zeros(4))


def test_one_long_tile_many_lanes():
    # reference tests/test_executor.py:145-155: 100 atoms in one tile, 8 lanes
    off = np.array([0, 100])
    y = oracle.spmv(off, np.zeros(100, np.int64), np.ones(100), np.ones(1), "merge-path", lanes=8)
    assert y[0] == 100.0
    la, al, at = oracle.assignment(off, "merge-path", 8)
    assert la.sum() == 100 and (la > 0).sum() >= 2 and (at == 0).all()


def test_abs_row_sums_and_tolerance():
    off, col, val = [0, 2, 3], [0, 1, 1], [1.0, -2.0, 3.0]
    s = oracle.abs_row_sums(off, col, val, np.array([1.0, 2.0]))
    np.testing.assert_array_equal(s, [5.0, 6.0])
    assert oracle.tolerance_ok([1.0], np.array([1.0 + 1e-6]), [1.0], 1e-5)[0]
    assert not oracle.tolerance_ok([1.0], np.array([1.0 + 1e-4]), [1.0], 1e-5)[0]


@pytest.mark.parametrize("threads", [1, 3])
def test_spmm_matches_reference(golden, threads):
    """C oracle SpMM vs lanework.spmm (numba) on every golden case (kernels.py:129-175)."""
    g = golden["spmm"]
    cases = list(golden.spmm_cases())
    for ck, (mi, ci, integer) in enumerate(g["meta"]):
        _, off, col, val, B, rows, cols = cases[mi]
        C = oracle.spmm(off, col, val, B, str(g["cfg_kind"][ci]), lanes=int(g["cfg_lanes"][ci]),
                        threads=threads, group_size=int(g["cfg_gs"][ci]),
                        tiles_per_block=int(g["cfg_tpb"][ci]))
        want = unpack(g["C"], g["C_idx"], ck).reshape(rows, B.shape[1])
        if integer:
            np.testing.assert_array_equal(C, want)
        else:
            assert oracle.tolerance_ok(C, want, oracle.abs_spmm_sums(off, col, val, B), 1e-12)[0]


def test_spmm_column_slices_equal_spmv():
    """column c of spmm(m, B) equals spmv(m, B[:, c]) exactly (integer data)."""
    rng = np.random.default_rng(5)
    off = np.concatenate([[0], np.cumsum(rng.integers(0, 9, size=40))])
    col = rng.integers(0, 30, size=int(off[-1]))
    val = rng.integers(-4, 5, size=col.size).astype(np.float64)
    B = rng.integers(-3, 4, size=(30, 6)).astype(np.float64)
    for kind in KIND_NAMES:
        C = oracle.spmm(off, col, val, B, kind, lanes=7)
        for c in range(6):
            np.testing.assert_array_equal(C[:, c], oracle.spmv(off, col, val, B[:, c], kind, lanes=7))


def test_traversal_oracle_matches_reference(golden):
    """Oracle frontier SSSP/BFS == lanework.sssp / bfs == dijkstra / serial_bfs, bit for bit."""
    g = golden["traversal"]
    for k, src in enumerate(g["src"]):
        off, col = unpack(g["off"], g["off_idx"], k), unpack(g["col"], g["col_idx"], k)
        w = unpack(g["w"], g["col_idx"], k)
        dist = oracle.sssp(off, col, w, int(src))
        np.testing.assert_array_equal(dist, unpack(g["dist"], g["v_idx"], k))
        np.testing.assert_array_equal(dist, unpack(g["dijkstra"], g["v_idx"], k))
        depth = oracle.bfs(off, col, int(src))
        np.testing.assert_array_equal(depth, unpack(g["depth"], g["v_idx"], k))
        np.testing.assert_array_equal(depth, unpack(g["serial_bfs"], g["v_idx"], k))
