"""Host-side API of the package against the reference: names, signatures,
error behaviour and golden vectors (CPU only; mirrors the reference's
test_schedules.py / test_work.py / test_executor.py)."""

import itertools
from collections import Counter

import numpy as np
import pytest

from conftest import unpack

import paper_2301_04792_b200 as lw
from paper_2301_04792_b200 import ScheduleKind


def ts_(offsets):
    return lw.TileSet(np.asarray(offsets, dtype=np.int64))


# ---- work domain (reference tests/test_work.py) ------------------------------------------

def test_tile_set_basics():
    m = lw.CsrMatrix(3, 3, [0, 2, 3, 6], [0, 1, 2, 0, 1, 2], [1.0] * 6)
    ts = lw.csr_tile_set(m)
    assert (ts.num_tiles, ts.num_atoms) == (3, 6)
    assert [ts.atoms_in_tile(t) for t in range(3)] == [2, 1, 3]
    assert [ts.atom_offset(t) for t in range(4)] == [0, 2, 3, 6]
    assert list(ts.atoms(2)) == [3, 4, 5]
    with pytest.raises(ValueError):
        lw.TileSet([1, 2])
    with pytest.raises(ValueError):
        lw.TileSet([0, 3, 2])
    with pytest.raises(ValueError):
        lw.TileSet([])


def test_ranges():
    assert list(lw.step_range(0, 10, 3)) == [0, 3, 6, 9]
    assert list(lw.step_range(7, 3, 2)) == []
    with pytest.raises(ValueError):
        lw.step_range(0, 10, 0)
    assert list(lw.lane_stride_range(1, 4, 10)) == [1, 5, 9]
    with pytest.raises(ValueError):
        lw.lane_stride_range(4, 4, 10)
    with pytest.raises(ValueError):
        lw.lane_stride_range(0, 0, 10)
    for p, n in [(4, 10), (1, 7), (13, 5), (64, 10_000)]:
        got = sorted(itertools.chain.from_iterable(lw.lane_stride_range(l, p, n) for l in range(p)))
        assert got == list(range(n))
    assert list(itertools.islice(lw.infinite_range(5), 4)) == [5, 6, 7, 8]


# ---- schedules (reference tests/test_schedules.py) ------------------------------------------

def test_schedule_kind_names_and_aliases():
    assert ScheduleKind("merge-path") is ScheduleKind.MERGE_PATH
    assert ScheduleKind.WORK_ORIENTED is ScheduleKind.MERGE_PATH
    assert ScheduleKind("work_oriented") is ScheduleKind.MERGE_PATH
    assert ScheduleKind("thread_mapped") is ScheduleKind.THREAD_MAPPED
    assert [k.value for k in ScheduleKind] == ["thread-mapped", "merge-path", "group-mapped"]
    with pytest.raises(ValueError):
        ScheduleKind("nope")


def test_merge_path_known_answers():
    ts = ts_([0, 2, 3, 6])
    assert lw.merge_path_search(0, ts) == (0, 0)
    assert lw.merge_path_search(9, ts) == (3, 6)
    assert lw.merge_path_search(3, ts) == (1, 2)
    with pytest.raises(ValueError):
        lw.merge_path_search(-1, ts_([0, 2]))
    with pytest.raises(ValueError):
        lw.merge_path_search(4, ts_([0, 2]))
    np.testing.assert_array_equal(lw.merge_path_partition(ts, 1), [[0, 0], [3, 6]])
    np.testing.assert_array_equal(lw.merge_path_partition(ts, 3), [[0, 0], [1, 2], [2, 4], [3, 6]])
    work = np.diff(lw.merge_path_partition(ts_([0, 1]), 8), axis=0).sum(axis=1)
    assert work.sum() == 2 and np.all(work[2:] == 0)
    with pytest.raises(ValueError):
        lw.merge_path_partition(ts, 0)


def test_merge_path_matches_golden(golden):
    g = golden["schedules"]
    k = 0
    for s, off in enumerate(golden.tile_sets()):
        ts = lw.TileSet(off)
        want = unpack(g["search"], g["search_idx"], s).reshape(-1, 2)
        got = np.array([tuple(lw.merge_path_search(d, ts)) for d in range(want.shape[0])])
        np.testing.assert_array_equal(got.reshape(-1, 2), want)
        for p in g["lane_counts"]:
            np.testing.assert_array_equal(lw.merge_path_partition(ts, int(p)),
                                          unpack(g["parts"], g["parts_idx"], k).reshape(-1, 2))
            sl = lw.merge_path_slices(ts, int(p))
            for a, b in zip(sl, sl[1:]):
                assert (a.tile_end, a.atom_end) == (b.tile_begin, b.atom_begin)
            k += 1


def test_prefix_sum():
    np.testing.assert_array_equal(lw.exclusive_prefix_sum([]), [0])
    np.testing.assert_array_equal(lw.exclusive_prefix_sum([2, 1, 3]), [0, 2, 3, 6])
    with pytest.raises(OverflowError):
        lw.exclusive_prefix_sum([1 << 62, 1 << 62, 1 << 62])
    with pytest.raises(ValueError):
        lw.exclusive_prefix_sum([1, -2, 3])


def test_group_plan_and_get_tile_known_answers():
    plan = lw.group_plan(ts_([0, 2, 3, 6]), 0, 1, tiles_per_block=3)
    assert (plan.tile_begin, plan.tile_count, plan.total_atoms) == (0, 3, 6)
    np.testing.assert_array_equal(plan.prefix, [0, 2, 3, 6])
    np.testing.assert_array_equal(lw.group_plan(ts_([0, 0, 0]), 0, 1, 2).prefix, [0, 0, 0])
    ts = ts_([0, 1, 2, 3, 4])
    with pytest.raises(ValueError):
        lw.group_plan(ts, 2, 2, 1)
    with pytest.raises(ValueError):
        lw.group_plan(ts, 0, 2, 1, block=1)
    assert lw.group_plan(ts, 1, 2, 1, block=3).tile_begin == 3
    p = lw.GroupPlan(0, 3, np.array([0, 2, 3, 6]))
    assert [lw.get_tile(p, a) for a in (4, 0, 2)] == [2, 0, 1]
    assert lw.get_tile(lw.GroupPlan(0, 2, np.array([0, 0, 5])), 0) == 1
    with pytest.raises(ValueError):
        lw.get_tile(lw.GroupPlan(0, 1, np.array([0, 3])), 3)


def test_group_plan_get_tile_golden(golden):
    g = golden["schedules"]
    k = 0
    for off in golden.tile_sets():
        ts = lw.TileSet(off)
        for tpb in (1, 3, 32):
            nb = lw.num_blocks(ts, tpb)
            for b in range(nb):
                plan = lw.group_plan(ts, b, nb, tpb, block=b)
                np.testing.assert_array_equal(plan.prefix, unpack(g["plans"], g["plans_idx"], k))
                want = unpack(g["tiles"], g["tiles_idx"], k)
                got = [lw.get_tile(plan, a) for a in range(plan.total_atoms)]
                np.testing.assert_array_equal(got, want)
                k += 1


# ---- executor (reference tests/test_executor.py) -----------------------------------------

def test_executor_config_validation():
    c = lw.ExecutorConfig()
    # the reference resolves lanes=None to worker_threads*32 (executor.py:54-55)
    assert c.schedule is ScheduleKind.MERGE_PATH and c.lanes == 32 and c.lane_count == 32
    assert c.lanes_auto   # ... and the GPU launch is sized for the device
    assert c.tiles_per_block == 32 and c.group_count == 1
    assert lw.ExecutorConfig(worker_threads=4).lanes == 128
    explicit = lw.ExecutorConfig(lanes=32)
    assert explicit.lanes == 32 and not explicit.lanes_auto
    import dataclasses
    assert not dataclasses.replace(c, lanes=64).lanes_auto
    assert lw.ExecutorConfig(schedule="work-oriented").schedule is ScheduleKind.MERGE_PATH
    for bad in (dict(worker_threads=0), dict(lanes=0), dict(group_size=0),
                dict(tiles_per_block=0)):
        with pytest.raises(ValueError):
            lw.ExecutorConfig(**bad)
    c = lw.ExecutorConfig(lanes=10, group_size=4)
    assert c.group_count == 3 and list(c.group_lanes(2)) == [8, 9]


def test_imbalance_matches_golden(golden):
    g = golden["schedules"]
    shapes = g["gm_shapes"]
    k = 0
    kinds = list(ScheduleKind)[:3]
    for off in golden.tile_sets():
        ts = lw.TileSet(off)
        for p in g["lane_counts"]:
            for kind in kinds:
                for gs, tpb in (shapes if kind is ScheduleKind.GROUP_MAPPED else [(32, 32)]):
                    cfg = lw.ExecutorConfig(schedule=kind, lanes=int(p), group_size=int(gs),
                                            tiles_per_block=int(tpb))
                    np.testing.assert_array_equal(lw.imbalance(ts, cfg).per_lane_atoms,
                                                  unpack(g["imbal"], g["imbal_idx"], k))
                    k += 1


def test_imbalance_known_answers():
    ts = ts_([0, 1000] + [1000] * 7)
    r = lw.imbalance(ts, lw.ExecutorConfig(schedule=ScheduleKind.THREAD_MAPPED, lanes=8))
    assert r.imbalance_factor == pytest.approx(8.0) and r.per_lane_atoms.sum() == 1000
    r = lw.imbalance(ts_([0, 1000]), lw.ExecutorConfig(schedule=ScheduleKind.MERGE_PATH, lanes=8))
    assert r.max <= -(-1001 // 8)
    r = lw.imbalance(ts_([0, 0, 0]), lw.ExecutorConfig(lanes=4))
    assert r.imbalance_factor == 1.0


def _visits(ts, cfg):
    got = {}
    if cfg.schedule is ScheduleKind.MERGE_PATH:
        def atom_fn(lane, tile, atom):
            got.setdefault(atom, []).append((lane, tile))
            return 0.0

        lw.execute_merge_path(cfg, ts, atom_fn, lambda *a: None)
    else:
        def work_fn(lane, tile, atoms):
            for a in atoms:
                got.setdefault(a, []).append((lane, tile))

        lw.execute_tile_major(cfg, ts, work_fn)
    return got


def test_walkers_and_schedule_objects_match_reference_assignment(golden):
    g = golden["schedules"]
    sets = golden.tile_sets()
    kinds = list(ScheduleKind)[:3]
    for k, (si, p, ki, gs, tpb) in enumerate(g["assign_meta"]):
        ts = lw.TileSet(sets[si])
        cfg = lw.ExecutorConfig(schedule=kinds[ki], lanes=int(p), group_size=int(gs),
                                tiles_per_block=int(tpb))
        want_lane = unpack(g["assign_lane"], g["assign_idx"], k)
        want_tile = unpack(g["assign_tile"], g["assign_idx"], k)
        got = _visits(ts, cfg)
        assert all(len(v) == 1 for v in got.values()) and len(got) == ts.num_atoms
        for a in range(ts.num_atoms):
            assert got[a][0] == (want_lane[a], want_tile[a])
        sched = lw.make_schedule(ts, cfg)
        seen = Counter()
        for lane, tile, atom in sched.assignment():
            assert (lane, tile) == (want_lane[atom], want_tile[atom])
            seen[atom] += 1
        assert seen == Counter(range(ts.num_atoms))


def test_merge_path_executor_carries():
    ts = ts_([0, 2, 3, 6])
    cfg = lw.ExecutorConfig(schedule=ScheduleKind.MERGE_PATH, lanes=3)
    done = []
    carries = lw.execute_merge_path(cfg, ts, lambda lane, t, a: float(a),
                                    lambda lane, t, acc: done.append((lane, t, acc)))
    assert done == [(0, 0, 1.0), (1, 1, 2.0), (2, 2, 9.0)]
    assert carries[0].tile == lw.SENTINEL_TILE and carries[1] == (2, 3.0)
    best = np.zeros(2)
    vals = np.array([3.0, 9.0, 1.0, 4.0, 8.0, 2.0, 6.0])
    carries = lw.execute_merge_path(
        lw.ExecutorConfig(schedule=ScheduleKind.MERGE_PATH, lanes=3), ts_([0, 4, 7]),
        lambda lane, t, a: vals[a], lambda lane, t, acc: best.__setitem__(t, max(best[t], acc)),
        carry_policy=lw.CarryPolicy(identity=0.0, combine=max))
    lw.fixup_combine(carries, lambda t, p: best.__setitem__(t, max(best[t], p)))
    np.testing.assert_array_equal(best, [9.0, 8.0])
    with pytest.raises(ValueError):
        lw.execute_tile_major(cfg, ts, lambda *a: None)
    with pytest.raises(ValueError):
        lw.execute_merge_path(lw.ExecutorConfig(schedule=ScheduleKind.THREAD_MAPPED), ts,
                              lambda *a: 0.0, lambda *a: None)


# ---- data + generators (reference tests/test_sparse.py) ----------------------------------

def test_generators_match_reference_golden(golden):
    gen = golden["generators"]
    for c in range(int(gen["count"])):
        a = gen[f"c{c}_args"]
        if str(gen[f"c{c}_kind"]) == "random":
            m = lw.generate_random_csr(int(a[0]), int(a[1]), int(a[2]), int(a[3]))
        else:
            m = lw.generate_power_law_csr(int(a[0]), float(a[1]), float(a[2]), int(a[3]))
        np.testing.assert_array_equal(m.row_offsets, gen[f"c{c}_off"])
        np.testing.assert_array_equal(m.col_indices, gen[f"c{c}_col"])
        np.testing.assert_array_equal(m.values, gen[f"c{c}_val"])
        lw.validate_csr(m)


def test_generator_errors_and_validate():
    with pytest.raises(ValueError):
        lw.generate_random_csr(2, 2, 5, seed=0)
    for bad in [(0, 1.0, 1.0), (5, 0.0, 1.0), (5, 1.0, 0.0)]:
        with pytest.raises(ValueError):
            lw.generate_power_law_csr(*bad, seed=0)
    with pytest.raises(ValueError):
        lw.validate_csr(lw.CsrMatrix(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0]))
    with pytest.raises(ValueError):
        lw.validate_csr(lw.CsrMatrix(1, 2, [0, 2], [1, 0], [1.0, 1.0]))
    with pytest.raises(ValueError):
        lw.validate_csr(lw.CsrMatrix(1, 2, [0, 1], [2], [1.0]))
    lw.validate_csr(lw.CsrMatrix(2, 2, [0, 1, 2], [1, 0], [1.0, 1.0]))


def test_banded_and_stats():
    m = lw.generate_banded_csr(1000, 16, seed=2)
    lw.validate_csr(m)
    assert m.nnz == 1000 * 33 - 2 * sum(range(1, 17))
    st = lw.row_length_stats(m.row_offsets)
    assert st["max"] == 33 and st["empty_rows"] == 0
    assert abs(lw.generate_banded_csr(1_000_000, 16, 2).nnz - 32_999_728) == 0


def test_heuristic_dispatch():
    # reference acceptance criterion 6 (tests/test_acceptance.py:201-211)
    assert lw.choose_spmv_schedule(400, 400, 5000) is ScheduleKind.THREAD_MAPPED
    assert lw.choose_spmv_schedule(10**5, 10**5, 10**6) is ScheduleKind.MERGE_PATH
    for rows, cols, nnz in itertools.product(range(498, 503), range(498, 503), range(9998, 10003)):
        want = (ScheduleKind.THREAD_MAPPED if (rows < 500 or cols < 500) and nnz < 10000
                else ScheduleKind.MERGE_PATH)
        assert lw.choose_spmv_schedule(rows, cols, nnz) is want
    with pytest.raises(ValueError):
        lw.HeuristicConfig(alpha=0)


def test_backend_seam_has_no_cpu_fallback(monkeypatch):
    assert lw.backend_name() == "cuda" and not lw.numba_active()
    with pytest.raises(ValueError):
        with lw.use_backend("numpy"):
            pass
    with lw.use_backend("cuda"):
        assert lw.cuda_active()
    import torch

    if not torch.cuda.is_available():
        m = lw.CsrMatrix(2, 2, [0, 2, 3], [0, 1, 1], [1.0, 2.0, 3.0])
        with pytest.raises(lw.BackendUnavailable):
            lw.spmv(m, np.ones(2))


def test_atomic_min_array_semantics():
    """executor.AtomicMinArray (reference executor.py:254-283)."""
    import paper_2301_04792_b200 as lwb

    a = lwb.AtomicMinArray(np.array([np.inf, 2.0]))
    assert a.atomic_min(0, 3.0) == np.inf and a.values[0] == 3.0
    assert lwb.atomic_min_real(a, 1, 5.0) == 2.0 and a.values[1] == 2.0
    with pytest.raises(ValueError):
        a.atomic_min(0, -1.0)
    with pytest.raises(ValueError):
        lwb.AtomicMinArray(np.array([-1.0]))


# the reference's public names (lanework/__init__.py:65-122), all of which must exist here
REFERENCE_ALL = [
    "AtomicMinArray", "CarryOut", "CarryPolicy", "CooMatrix", "CsrMatrix", "ExecutorConfig",
    "Graph", "GroupPlan", "HeuristicConfig", "ImbalanceReport", "MatrixMarketError",
    "MergePathCoord", "MergePathSlice", "NUMBA_AVAILABLE", "SENTINEL_TILE",
    "ScheduleKind", "SsspState", "TileSet", "UNREACHED", "atomic_min_real", "backend_name", "bfs",
    "choose_spmv_schedule", "coo_to_csr", "csr_tile_set", "csr_to_coo", "exclusive_prefix_sum",
    "execute_merge_path", "execute_tile_major", "fixup_combine", "generate_power_law_csr",
    "generate_random_csr", "get_tile", "group_plan", "imbalance", "infinite_range",
    "lane_stride_range", "load_matrix_market", "merge_path_partition", "merge_path_search",
    "merge_path_slices", "numba_active", "parse_matrix_market", "spmm", "spmv", "spmv_auto",
    "sssp", "sssp_init", "sssp_pass", "step_range", "thread_mapped_tiles", "transpose_csr",
    "use_backend", "validate_coo", "validate_csr", "write_matrix_market",
]


def test_reference_public_names_exist():
    import paper_2301_04792_b200 as lwb

    missing = [n for n in REFERENCE_ALL if not hasattr(lwb, n)]
    assert not missing, missing
