"""GPU parity suite: the sm_100a kernels (through the C ABI) against the reference.

Every check compares the CUDA path with (a) golden vectors recorded from the
reference itself (tests/golden) or (b) the C oracle on the same seeded inputs:
  * schedule maps are bit-exact: merge-path partitions, group-plan prefixes,
    per-lane atom counts (== executor.imbalance) and the (lane, tile) each atom
    is processed by (== the reference executors), each atom exactly once;
  * y is bit-exact on integer-valued data (fp32 and fp64, every schedule);
  * otherwise |y - y_ref| <= rtol * sum_j |A_ij x_j| with rtol 1e-5 (fp32) and
    1e-12 (fp64), the north star's tolerance (BASELINE.json).
"""

import dataclasses

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
    off = np.asarray(off, np.int64)
    odt = torch.int32 if offset_bits == 32 else torch.int64
    return DeviceCsr(len(off) - 1, int(cols),
                     torch.as_tensor(off).to("cuda", odt),
                     torch.as_tensor(np.asarray(col, np.int64)).to("cuda", torch.int32),
                     torch.as_tensor(np.asarray(val, np.float64)).to("cuda", dtype))


def run(m, x, kind, lanes=None, gs=32, tpb=None):
    cfg = ExecutorConfig(schedule=KINDS[kind] if isinstance(kind, str) else kind, lanes=lanes,
                         group_size=gs, tiles_per_block=tpb)
    xt = torch.as_tensor(np.asarray(x, np.float64)).to("cuda", m.dtype)
    return lwb.spmv(m, xt, cfg).double().cpu().numpy()


def check_tol(y, off, col, val, x, dtype, y_ref=None):
    if y_ref is None:
        y_ref = oracle.spmv(off, col, val, x, "thread-mapped", lanes=1)
    scale = oracle.abs_row_sums(off, col, val, x)
    ok, worst = oracle.tolerance_ok(y, y_ref, scale, RTOL[dtype])
    assert ok, f"tolerance exceeded: worst err/bound = {worst:.3g}"


# ---- schedule maps (bit-exact) ----------------------------------------------------------

@pytest.mark.parametrize("bits", [32, 64])
def test_partition_matches_reference_golden(golden, bits):
    g = golden["schedules"]
    sets = golden.tile_sets()
    lane_counts = list(g["lane_counts"])
    k = 0
    for off in sets:
        odt = torch.int32 if bits == 32 else torch.int64
        m = DeviceCsr(len(off) - 1, 1, torch.as_tensor(off).to("cuda", odt),
                      torch.zeros(int(off[-1]), dtype=torch.int32, device="cuda"),
                      torch.zeros(int(off[-1]), dtype=torch.float32, device="cuda"))
        for p in lane_counts:
            want = unpack(g["parts"], g["parts_idx"], k).reshape(-1, 2)
            got = lwb.device_merge_path_partition(m, int(p)).cpu().numpy()
            np.testing.assert_array_equal(got, want)
            k += 1


def test_partition_every_diagonal_matches_reference_search(golden):
    """lanes = total makes every diagonal a split point: the full search table."""
    g = golden["schedules"]
    for s, off in enumerate(golden.tile_sets()):
        want = unpack(g["search"], g["search_idx"], s).reshape(-1, 2)
        total = len(off) - 1 + int(off[-1])
        if total == 0:
            continue
        m = DeviceCsr(len(off) - 1, 1, torch.as_tensor(off).to("cuda", torch.int32),
                      torch.zeros(int(off[-1]), dtype=torch.int32, device="cuda"),
                      torch.zeros(int(off[-1]), dtype=torch.float32, device="cuda"))
        got = lwb.device_merge_path_partition(m, total).cpu().numpy()
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("bits", [32, 64])
def test_partition_both_search_paths_match_oracle(bits):
    """Partitions of <= 12288 boundaries take the warp-cooperative search, larger
    ones the per-thread binary search (spmv_work_oriented.cu launch_search): both
    sides of the threshold against the oracle's search (reference
    schedules.py:63-110) on a skewed matrix with runs of empty rows and one row
    of 300 K atoms."""
    rng = np.random.default_rng(11)
    lengths = np.minimum(rng.zipf(1.4, 200_000) - 1, 5000)
    lengths[50_000:90_000] = 0
    lengths[120_000] = 300_000
    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    nnz = int(off[-1])
    odt = torch.int32 if bits == 32 else torch.int64
    m = DeviceCsr(len(off) - 1, 1, torch.as_tensor(off).to("cuda", odt),
                  torch.zeros(nnz, dtype=torch.int32, device="cuda"),
                  torch.zeros(nnz, dtype=torch.float32, device="cuda"))
    for p in (1, 7, 4096, 12287, 12288, 12289, 30_000):
        want = oracle.merge_path_partition(off, p, threads=4)
        got = lwb.device_merge_path_partition(m, p).cpu().numpy()
        np.testing.assert_array_equal(got, want, err_msg=f"lanes={p}")


def test_group_plan_prefix_matches_reference_golden(golden):
    g = golden["schedules"]
    k = 0
    for off in golden.tile_sets():
        ts = lwb.TileSet(off)
        for tpb in (1, 3, 32):
            nb = lwb.num_blocks(ts, tpb)
            if nb == 0:
                continue
            got = lwb.device_group_plan_prefix(ts, tpb, device="cuda").cpu().numpy()
            for b in range(nb):
                want = unpack(g["plans"], g["plans_idx"], k)
                np.testing.assert_array_equal(got[b, :len(want)], want)
                assert (got[b, len(want):] == want[-1]).all()
                k += 1


def test_probe_assignment_matches_reference_executors(golden):
    """Per-atom (lane, tile) and per-lane counts of the instrumented kernels equal
    what the reference executors hand out (execute_tile_major/execute_merge_path)."""
    g = golden["schedules"]
    sets = golden.tile_sets()
    kinds = list(ScheduleKind)[:3]
    for k, (si, p, ki, gs, tpb) in enumerate(g["assign_meta"]):
        off = sets[si]
        nnz = int(off[-1])
        if nnz == 0:
            continue
        m = DeviceCsr(len(off) - 1, 1, torch.as_tensor(off).to("cuda", torch.int32),
                      torch.zeros(nnz, dtype=torch.int32, device="cuda"),
                      torch.ones(nnz, dtype=torch.float64, device="cuda"))
        cfg = ExecutorConfig(schedule=kinds[ki], lanes=int(p), group_size=int(gs),
                             tiles_per_block=int(tpb))
        x = torch.ones(1, dtype=torch.float64, device="cuda")
        y, pr, lanes = lwb.spmv_probe(m, x, cfg)
        np.testing.assert_array_equal(pr["atom_visits"], np.ones(nnz))
        np.testing.assert_array_equal(pr["atom_lane"], unpack(g["assign_lane"], g["assign_idx"], k))
        np.testing.assert_array_equal(pr["atom_tile"], unpack(g["assign_tile"], g["assign_idx"], k))
        np.testing.assert_array_equal(y.cpu().numpy(), np.diff(off).astype(np.float64))
        ref_counts = lwb.imbalance(lwb.TileSet(off), cfg).per_lane_atoms
        np.testing.assert_array_equal(pr["lane_atoms"], ref_counts)


@pytest.mark.parametrize("kind,gs", [("thread-mapped", 32), ("merge-path", 32),
                                     ("group-mapped", 32), ("group-mapped", 256),
                                     ("group-mapped", 128), ("group-mapped", 4)])
def test_probe_auto_lanes_matches_oracle(kind, gs):
    """At device-chosen lane counts (the production launch) the per-thread work
    equals the oracle's assignment for that P, on a skewed power-law matrix."""
    m = lwb.generate_power_law_csr(20000, 12.0, 1.2, seed=7)
    dm = m.to_device("float32")
    cfg = lwb.device_config(ExecutorConfig(schedule=KINDS[kind], group_size=gs), dm)
    x = torch.ones(m.cols, dtype=torch.float32, device="cuda")
    y, pr, lanes = lwb.spmv_probe(dm, x, cfg)
    la, al, at = oracle.assignment(m.row_offsets, kind, lanes, gs, gs)
    np.testing.assert_array_equal(pr["atom_visits"], np.ones(m.nnz))
    np.testing.assert_array_equal(pr["lane_atoms"], la)
    np.testing.assert_array_equal(pr["atom_lane"], al)
    np.testing.assert_array_equal(pr["atom_tile"], at)


# ---- y against the reference (golden) ------------------------------------------------------

@pytest.mark.parametrize("bits", [32, 64])
def test_spmv_fp64_matches_reference_golden(golden, bits):
    g = golden["spmv"]
    for (mi, ci, integer), yk in zip(g["meta"], range(len(g["meta"]))):
        k, off, col, val, x, rows, cols = list(golden.spmv_cases())[mi]
        want = unpack(g["y"], g["y_idx"], yk)
        m = dev_csr(off, col, val, cols, torch.float64, bits)
        kind = str(g["cfg_kind"][ci])
        lanes, gs, tpb = int(g["cfg_lanes"][ci]), int(g["cfg_gs"][ci]), int(g["cfg_tpb"][ci])
        y = run(m, x, kind, lanes, gs, tpb)
        general = kind == "group-mapped" and not (gs == tpb == 32 and lanes % 32 == 0) and not (
            gs == tpb and gs in (64, 128, 256) and lanes % gs == 0)
        if integer or general:
            # general group shapes sum each tile in the reference's member-major
            # order with unfused fp64 ops (k_group_tiles): bit-identical y
            np.testing.assert_array_equal(y, want, err_msg=f"{mi} {kind} lanes={lanes} gs={gs}")
        else:
            scale = oracle.abs_row_sums(off, col, val, x)
            ok, worst = oracle.tolerance_ok(y, want, scale, 1e-12)
            assert ok, (mi, kind, worst)


# ---- integer data: bit-exact across schedules, lane counts and dtypes ---------------------

@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_integer_bit_exact_all_schedules(dtype):
    """Acceptance criterion 4 (reference tests/test_acceptance.py:136-166) on the GPU."""
    rng = np.random.default_rng(88)
    cfgs = [("thread-mapped", None, 32), ("merge-path", None, 32), ("group-mapped", None, 32),
            ("group-mapped", None, 256), ("thread-mapped", 64, 32), ("merge-path", 64, 32),
            ("group-mapped", 64, 4), ("group-mapped", 64, 32), ("group-mapped", 64, 256),
            ("merge-path", 7, 32), ("group-mapped", None, 128), ("group-mapped", None, 64)]
    for _ in range(40):
        rows, cols = int(rng.integers(1, 513)), int(rng.integers(1, 513))
        nnz = int(rng.integers(0, min(8192, rows * cols) + 1))
        m = integer_csr(rng, rows, cols, nnz)
        x = rng.integers(-3, 4, size=cols).astype(np.float64)
        want = m.to_dense() @ x
        dm = m.to_device(dtype)
        for kind, lanes, gs in cfgs:
            np.testing.assert_array_equal(run(dm, x, kind, lanes, gs, gs), want,
                                          err_msg=f"{kind} lanes={lanes} gs={gs}")


# ---- fp32 tolerance on the north-star inputs -----------------------------------------------

@pytest.fixture(scope="module")
def c1():
    m = lwb.generate_random_csr(10_000, 10_000, 1_000_000, seed=1)
    vals32 = m.values.astype(np.float32).astype(np.float64)
    x = np.random.default_rng(42).random(m.cols).astype(np.float32).astype(np.float64)
    return m, vals32, x


@pytest.mark.parametrize("kind,gs", [("thread-mapped", 32), ("merge-path", 32),
                                     ("group-mapped", 32), ("group-mapped", 256)])
def test_c1_fp32_within_tolerance(c1, kind, gs):
    m, vals32, x = c1
    dm = m.to_device("float32")
    y = run(dm, x, kind, None, gs, gs)
    check_tol(y, m.row_offsets, m.col_indices, vals32, x, torch.float32)


@pytest.mark.parametrize("skew", [3.0, 1.5, 1.1])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_power_law_sweep_within_tolerance(skew, dtype):
    m = lwb.generate_power_law_csr(1 << 16, 16.0, skew, seed=4)
    vals = m.values.astype(np.float32).astype(np.float64) if dtype == torch.float32 else m.values
    x = np.random.default_rng(42).random(m.cols)
    x = x.astype(np.float32).astype(np.float64) if dtype == torch.float32 else x
    dm = m.to_device(dtype)
    y_ref = oracle.spmv(m.row_offsets, m.col_indices, vals, x, "merge-path", threads=4)
    for kind, gs in [("thread-mapped", 32), ("merge-path", 32), ("group-mapped", 32),
                     ("group-mapped", 256)]:
        check_tol(run(dm, x, kind, None, gs, gs), m.row_offsets, m.col_indices, vals, x, dtype,
                  y_ref)


def test_all_positive_long_rows_fp32():
    """one fp32 accumulator fails 1e-5 at 7e5 positive terms;
    fp64 accumulation keeps every schedule inside the bound."""
    rows, per = 4, 700_000
    off = np.arange(rows + 1, dtype=np.int64) * per
    rng = np.random.default_rng(3)
    col = np.tile(np.arange(per, dtype=np.int64), rows)
    val = rng.random(rows * per).astype(np.float32).astype(np.float64)
    x = rng.random(per).astype(np.float32).astype(np.float64)
    m = dev_csr(off, col, val, per, torch.float32)
    for kind in ("thread-mapped", "merge-path", "group-mapped"):
        check_tol(run(m, x, kind), off, col, val, x, torch.float32)


@pytest.mark.parametrize("gs", [256, 128, 64, 32])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_group_tiles_long_row_runs(gs, dtype):
    """Blocks whose iterations fall inside one long row (the block tile's
    single-tile path): runs starting and ending on iteration boundaries, runs
    broken by short rows, one row spanning many iterations, empty rows between.
    Integer data bit-exact against the oracle, float data within the bound and
    bit-identical from run to run."""
    rng = np.random.default_rng(21)
    lens = rng.integers(0, 6, size=3 * gs)
    lens[[0, 3, 5, gs - 1, gs, gs + 2]] = [5000, 1024, 1025, 4 * 1024 * (gs // 64 or 1), 2048, 100_000]
    lens[gs + 1] = 0
    cols = 5000
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = np.concatenate([np.sort(rng.choice(cols, size=int(n), replace=n > cols)) for n in lens if n])
    for integer in (True, False):
        val = (rng.integers(-3, 4, size=col.size).astype(np.float64) if integer
               else rng.random(col.size) * 2 - 1)
        x = rng.integers(-3, 4, size=cols).astype(np.float64) if integer else rng.random(cols)
        if dtype == torch.float32:
            val, x = val.astype(np.float32).astype(np.float64), x.astype(np.float32).astype(np.float64)
        m = dev_csr(off, col, val, cols, dtype)
        y = run(m, x, "group-mapped", None, gs, gs)
        if integer:
            np.testing.assert_array_equal(y, oracle.spmv(off, col, val, x, "thread-mapped", lanes=1))
        else:
            check_tol(y, off, col, val, x, dtype)
            np.testing.assert_array_equal(y, run(m, x, "group-mapped", None, gs, gs))


# ---- edge cases the reference tests -------------------------------------------------------

@pytest.mark.parametrize("kind", ["thread-mapped", "merge-path", "group-mapped"])
def test_edge_cases(kind):
    cases = [
        ([0, 0, 0, 0], [], [], 3),                 # all rows empty
        ([0, 1], [0], [2.5], 1),                   # single atom
        ([0, 2, 3], [0, 1, 1], [1.0, 2.0, 3.0], 2),  # reference 2x2 example -> [3, 3] with x=1
        ([0, 0, 5, 5, 5], [0, 1, 2, 3, 4], [1.0] * 5, 5),
    ]
    for off, col, val, cols in cases:
        m = dev_csr(off, col, val, cols, torch.float64)
        x = np.ones(cols)
        want = np.zeros(len(off) - 1)
        for r in range(len(off) - 1):
            want[r] = sum(val[a] * x[col[a]] for a in range(off[r], off[r + 1]))
        for lanes in (None, 1, 2, 3, 100):
            np.testing.assert_array_equal(run(m, x, kind, lanes), want)


def test_dimension_mismatch_raises():
    m = dev_csr([0, 1, 2], [0, 1], [1.0, 1.0], 2)
    with pytest.raises(ValueError):
        lwb.spmv(m, torch.ones(3, dtype=torch.float64, device="cuda"))
    host = lwb.CsrMatrix(3, 3, np.arange(4), np.arange(3), np.ones(3))
    with pytest.raises(ValueError):
        lwb.spmv(host, np.ones(4))


def test_host_operands_match_reference_api():
    """spmv(CsrMatrix, ndarray) returns a float64 ndarray like the reference."""
    m = lwb.CsrMatrix(2, 2, [0, 2, 3], [0, 1, 1], [1.0, 2.0, 3.0])
    y = lwb.spmv(m, np.ones(2))
    assert isinstance(y, np.ndarray) and y.dtype == np.float64
    np.testing.assert_array_equal(y, [3.0, 3.0])
    ident = lwb.CsrMatrix(6, 6, np.arange(7), np.arange(6), np.ones(6))
    x = np.random.default_rng(0).random(6)
    np.testing.assert_array_equal(lwb.spmv(ident, x), x)
    for kind in ScheduleKind:
        np.testing.assert_array_equal(lwb.spmv(ident, x, ExecutorConfig(schedule=kind, lanes=3)), x)


@pytest.mark.parametrize("lanes", [None, 1, 3, 64, 1000])
def test_one_giant_row_carries(lanes):
    """One 3M-atom tile cut into many lanes/CTAs: ordered carry fix-up
    (reference test_executor.py:145-155 at GPU scale)."""
    n = 3_000_000
    off = np.array([0, 5, n - 7, n - 7, n], np.int64)
    col = np.concatenate([np.arange(5), np.arange(n - 12) % 1000, np.arange(7)])
    rng = np.random.default_rng(1)
    val = rng.integers(-3, 4, size=n).astype(np.float64)
    x = rng.integers(-3, 4, size=1000).astype(np.float64)
    m = dev_csr(off, col, val, 1000, torch.float64)
    want = oracle.spmv(off, col, val, x, "thread-mapped", lanes=1)
    np.testing.assert_array_equal(run(m, x, "merge-path", lanes), want)


def test_merge_path_run_to_run_deterministic():
    m = lwb.generate_power_law_csr(1 << 15, 32.0, 1.05, seed=9)
    dm = m.to_device("float32")
    x = torch.rand(m.cols, device="cuda")
    cfg = ExecutorConfig(schedule=ScheduleKind.MERGE_PATH)
    y0 = lwb.spmv(dm, x, cfg).clone()
    for _ in range(5):
        assert torch.equal(lwb.spmv(dm, x, cfg), y0)
    for kind, gs in [(ScheduleKind.GROUP_MAPPED, 32), (ScheduleKind.GROUP_MAPPED, 256),
                     (ScheduleKind.THREAD_MAPPED, 32)]:
        c = ExecutorConfig(schedule=kind, group_size=gs)
        a = lwb.spmv(dm, x, c).clone()
        assert torch.equal(lwb.spmv(dm, x, c), a)


# ---- generators ---------------------------------------------------------------------------

def test_rmat_device_matches_c_oracle():
    scale, ef, seed = 14, 16, 3
    th = lwb.rmat_thresholds()
    dm = lwb.generate_rmat_csr(scale, ef, seed, dtype="float64", chunk_edges=100_000)
    off, col, val = oracle.rmat_csr(scale, ef, seed, th, threads=4)
    np.testing.assert_array_equal(dm.row_offsets.cpu().numpy(), off)
    np.testing.assert_array_equal(dm.col_indices.cpu().numpy(), col)
    np.testing.assert_array_equal(dm.values.cpu().numpy(), val)


def test_banded_device_matches_host():
    host = lwb.generate_banded_csr(5000, 16, seed=2)
    dm = lwb.generate_banded_device(5000, 16, seed=2, dtype="float64")
    np.testing.assert_array_equal(dm.row_offsets.cpu().numpy(), host.row_offsets)
    np.testing.assert_array_equal(dm.col_indices.cpu().numpy(), host.col_indices)
    np.testing.assert_array_equal(dm.values.cpu().numpy(), host.values)


# ---- full-size property: C3 at a bounded scale ----------------------------------------------

@pytest.mark.parametrize("scale", [20])
def test_rmat_work_oriented_matches_oracle(scale):
    dm = lwb.generate_rmat_csr(scale, 16, seed=3, dtype="float32")
    x = torch.rand(dm.cols, device="cuda")
    y = lwb.spmv(dm, x, ExecutorConfig(schedule=ScheduleKind.WORK_ORIENTED)).double().cpu().numpy()
    off = dm.row_offsets.cpu().numpy().astype(np.int64)
    col = dm.col_indices.cpu().numpy().astype(np.int64)
    val = dm.values.cpu().numpy().astype(np.float64)
    xh = x.cpu().numpy().astype(np.float64)
    y_ref = oracle.spmv(off, col, val, xh, "merge-path", threads=oracle.default_threads())
    check_tol(y, off, col, val, xh, torch.float32, y_ref)


# ---- iterated SpMV (C5 shape, one GPU) ---------------------------------------------------

def test_power_iteration_single_gpu_matches_oracle():
    from paper_2301_04792_b200.distributed import RowShard, nnz_balanced_bounds, power_iteration

    dm = lwb.generate_rmat_csr(14, 16, seed=5, dtype="float64")
    off = dm.row_offsets.cpu().numpy().astype(np.int64)
    col = dm.col_indices.cpu().numpy().astype(np.int64)
    val = dm.values.cpu().numpy()
    shard = RowShard(nnz_balanced_bounds(off, 1), 0)
    cfg = ExecutorConfig(schedule=ScheduleKind.WORK_ORIENTED)
    x, norms = power_iteration(lambda v: lwb.spmv(dm, v, cfg), dm.rows, shard, 6,
                               dtype=torch.float64, device="cuda")
    xr = np.full(dm.rows, 1.0 / np.sqrt(dm.rows))
    ref_norms = []
    for _ in range(6):
        yr = oracle.spmv(off, col, val, xr, "merge-path", lanes=64)
        ref_norms.append(np.linalg.norm(yr))
        xr = yr / ref_norms[-1]
    np.testing.assert_allclose(norms, ref_norms, rtol=1e-10)
    np.testing.assert_allclose(x.cpu().numpy(), xr, rtol=1e-9, atol=1e-12)


def test_host_api_device_cache():
    """Host-API calls reuse the matrix's device copy while its arrays are unchanged;
    rebinding an array re-uploads; drop_device_cache forgets it."""
    from paper_2301_04792_b200.device import cached_device_csr, drop_device_cache

    m = lwb.generate_random_csr(200, 150, 2000, seed=3)
    x = np.random.default_rng(1).random(m.cols)
    y1 = lwb.spmv(m, x)
    d1 = cached_device_csr(m)
    assert cached_device_csr(m) is d1
    m.values = m.values * 2.0                      # rebinding: new upload, new result
    y2 = lwb.spmv(m, x)
    assert cached_device_csr(m) is not d1
    np.testing.assert_allclose(y2, 2.0 * y1, rtol=1e-12)
    m.values[:] = m.values / 2.0                   # in-place edit: outside the contract
    drop_device_cache(m)
    np.testing.assert_allclose(lwb.spmv(m, x), y1, rtol=1e-12)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_fused_power_iteration_matches_nccl_driver(dtype):
    """The SpMV-with-peer-writes path (world 1: the rank's own next-x buffer is
    its only peer) gives exactly the iterates of the plain SpMV driver."""
    from paper_2301_04792_b200.distributed import (RowShard, nnz_balanced_bounds, power_iteration,
                                                   power_iteration_fused)

    A = lwb.generate_rmat_csr(16, 8, seed=11, dtype="float32" if dtype == torch.float32 else "float64")
    shard = RowShard(nnz_balanced_bounds(A.row_offsets.cpu().numpy(), 1), 0)
    cfg = ExecutorConfig(schedule=ScheduleKind.MERGE_PATH)
    x1, n1 = power_iteration(lambda x: lwb.spmv(A, x, cfg), A.rows, shard, 6, dtype=dtype,
                             device="cuda")
    x2, n2 = power_iteration_fused(A, A.rows, shard, 6)
    torch.cuda.synchronize()
    assert torch.equal(x1, x2)
    assert n1 == n2


def test_peers_kernel_writes_every_buffer_at_the_row_base():
    """lw_spmv_work_oriented_peers: y plus every peer buffer get the shard's rows
    at row_base; rows outside the shard are untouched."""
    import ctypes

    from paper_2301_04792_b200 import _lib

    m = lwb.generate_power_law_csr(3000, 8.0, 1.2, seed=2)
    A = m.to_device("float32")
    x = torch.rand(A.cols, device="cuda")
    want = lwb.spmv(A, x, ExecutorConfig(schedule=ScheduleKind.MERGE_PATH))
    bufs = [torch.full((A.rows + 100,), -7.0, device="cuda") for _ in range(3)]
    y = torch.empty(A.rows, device="cuda")
    lib = _lib.load()
    need = lib.lw_spmv_work_oriented_workspace(A.rows, A.nnz, 0, _lib.LW_F32)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    ptrs = (ctypes.c_uint64 * 3)(*[b.data_ptr() for b in bufs])
    rc = lib.lw_spmv_work_oriented_peers(A.c_struct(), x.data_ptr(), y.data_ptr(), 0, ws.data_ptr(),
                                         need, 3, ptrs, 0, 60, torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    assert torch.equal(y, want)
    for b in bufs:
        assert torch.equal(b[60:60 + A.rows], want)
        assert (b[:60] == -7.0).all() and (b[60 + A.rows:] == -7.0).all()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_device_normalisation(dtype):
    """lw_vector_norm / lw_vector_scale: ||y|| within fp64 rounding of a sorted
    fp64 sum, run-to-run identical, x = y/||y||; y = 0 stays 0."""
    from paper_2301_04792_b200.distributed import _normalise

    g = torch.Generator(device="cuda").manual_seed(3)
    y = torch.randn(3_000_001, generator=g, device="cuda", dtype=dtype)
    n1, x1 = _normalise(y, dtype)
    n2, x2 = _normalise(y, dtype)
    assert torch.equal(n1, n2) and torch.equal(x1, x2)
    want = np.sqrt(np.sum(np.sort(y.double().cpu().numpy() ** 2)))
    assert abs(float(n1) - want) <= 1e-12 * want
    np.testing.assert_allclose(x1.double().cpu().numpy(), y.double().cpu().numpy() / want,
                               rtol=1e-6 if dtype == torch.float32 else 1e-14)
    z = torch.zeros(1000, device="cuda", dtype=dtype)
    nz, xz = _normalise(z, dtype)
    assert float(nz) == 0.0 and torch.equal(xz, z)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_group_general_shapes_deterministic(dtype):
    """General group shapes (no float atomics): repeated runs are bit-identical,
    with and without the probe, and equal the oracle's member-major sums."""
    m = lwb.generate_power_law_csr(20_000, 12.0, 1.2, seed=9)
    x = np.random.default_rng(5).random(m.cols)
    dm = m.to_device(dtype)
    xd = torch.as_tensor(x, device="cuda", dtype=dtype)
    scale = oracle.abs_row_sums(m.row_offsets, m.col_indices, m.values, x)
    for lanes, gs, tpb in [(96, 4, 4), (100, 32, 32), (1000, 256, 256), (512, 64, 7), (77, 5, 300)]:
        cfg = ExecutorConfig(schedule=ScheduleKind.GROUP_MAPPED, lanes=lanes, group_size=gs,
                             tiles_per_block=tpb)
        ys = [lwb.spmv(dm, xd, cfg) for _ in range(3)]
        assert all(torch.equal(ys[0], y) for y in ys[1:]), (lanes, gs, tpb)
        want = oracle.spmv(m.row_offsets, m.col_indices, m.values, x, "group-mapped", lanes=lanes,
                           group_size=gs, tiles_per_block=tpb)
        ok, worst = oracle.tolerance_ok(ys[0].double().cpu().numpy(), want, scale,
                                        1e-5 if dtype == torch.float32 else 1e-12)
        assert ok, (lanes, gs, tpb, worst)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_vector_scale_bit_exact_division(dtype):
    """lw_vector_scale equals (ValT)((double)y / nrm) bit for bit — for fp32 via the
    corrected reciprocal multiply (vector_ops.cu div_norm) — over random bit
    patterns covering every fp32 exponent (denormals, +-0, inf, NaN included),
    for norms from 2^-149 to 2^141, in place and out of place, odd lengths."""
    from paper_2301_04792_b200 import _lib
    from paper_2301_04792_b200.device import _dtype_code, current_stream

    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(11)
    n = (1 << 22) + 3
    if dtype == torch.float32:
        bits = torch.randint(-(1 << 31), 1 << 31, (n,), generator=g, device="cuda", dtype=torch.int64)
        y = bits.to(torch.int32).view(torch.float32)
        y[:4] = torch.tensor([0.0, -0.0, float("inf"), float("nan")], device="cuda")
    else:
        y = torch.randn(n, generator=g, device="cuda", dtype=dtype) * 1e3
    stream = current_stream(y.device)
    for b in (2.0 ** -149, 1e-30, 0.0071, 1.0 / 3.0, 1.0, 3.0, 1234.5678, 7.3e5, 1e30, 2.0 ** 141,
              float(torch.rand(1, generator=g, device="cuda")) * 1e4):
        nrm = torch.tensor(b, dtype=torch.float64, device="cuda")
        want = (y.double() / nrm).to(dtype)
        out = torch.empty_like(y)
        _lib.check(lib.lw_vector_scale(y.data_ptr(), n, _dtype_code(dtype), nrm.data_ptr(), out.data_ptr(),
                                       stream), "lw_vector_scale")
        yy = y.clone()
        _lib.check(lib.lw_vector_scale(yy.data_ptr(), n, _dtype_code(dtype), nrm.data_ptr(), yy.data_ptr(),
                                       stream), "lw_vector_scale")
        for got in (out, yy):
            iview = torch.int32 if dtype == torch.float32 else torch.int64
            same = (got.view(iview) == want.view(iview)) | (torch.isnan(got) & torch.isnan(want))
            assert bool(same.all()), f"norm {b}: {int((~same).sum())} elements differ"


def test_power_iteration_graph_replay_matches_eager():
    """The CUDA-graph-captured power iteration replays the exact eager iterates."""
    from paper_2301_04792_b200.distributed import (RowShard, nnz_balanced_bounds, power_iteration,
                                                   power_iteration_graph)

    A = lwb.generate_rmat_csr(15, 8, seed=5)
    shard = RowShard(nnz_balanced_bounds(A.row_offsets.cpu().numpy(), 1), 0)
    cfg = ExecutorConfig(schedule=ScheduleKind.MERGE_PATH)
    y = torch.empty(A.rows, dtype=A.dtype, device="cuda")

    def spmv(x):
        lwb.spmv(A, x, cfg, out=y)
        return y

    x1, n1 = power_iteration(spmv, A.rows, shard, 7, dtype=A.dtype, device="cuda")
    run = power_iteration_graph(spmv, A.rows, shard, 7, dtype=A.dtype, device="cuda")
    for _ in range(2):
        x2, n2 = run()
        torch.cuda.synchronize()
        assert torch.equal(x1, x2) and n1 == n2


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_group_warp_staged_and_cooperative_blocks_bit_exact(dtype):
    """Large enough for the staged/cooperative launch pair of the warp-tile kernel
    (>= 4 blocks per SM): short-row blocks (several shared-memory segments when a
    block holds more atoms than one segment), blocks with rows near the staged
    limit, and blocks with rows beyond it; integer data, so y is exact."""
    rng = np.random.default_rng(5)
    rows, cols = 40_000, 30_000
    lens = rng.integers(0, 41, size=rows)
    lens[::97] = rng.integers(100, 129, size=len(lens[::97]))
    lens[::1000] = 500
    lens[5000:5032] = 33   # one block of exactly 1056 atoms
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col = np.concatenate([np.sort(rng.choice(cols, size=int(n), replace=False)) for n in lens])
    val = rng.integers(-3, 4, size=len(col)).astype(np.float64)
    x = rng.integers(-3, 4, size=cols).astype(np.float64)
    want = oracle.spmv(off, col, val, x, "thread-mapped", lanes=1)
    m = dev_csr(off, col, val, cols, dtype)
    for lanes in (None, 32 * 700, 32 * 5000):
        np.testing.assert_array_equal(run(m, x, "group-mapped", lanes, 32, 32), want,
                                      err_msg=f"lanes={lanes}")


@pytest.mark.parametrize("kind,gs", [("thread-mapped", 32), ("merge-path", 32), ("group-mapped", 32),
                                     ("group-mapped", 256), ("group-mapped", 4)])
def test_debug_entry_points_match_the_probe(kind, gs):
    """lw_debug_lane_atom_counts / lw_debug_atom_tiles (SURVEY §8(b)'s named
    introspection calls) return what the probe records, and the per-lane counts
    equal the reference's imbalance() at the launch's lane count."""
    from paper_2301_04792_b200 import _lib
    from paper_2301_04792_b200.device import current_stream

    m = lwb.generate_power_law_csr(3000, 9.0, 1.3, seed=4)
    dm = m.to_device("float64")
    x = torch.as_tensor(np.random.default_rng(1).random(m.cols), device="cuda")
    cfg = ExecutorConfig(schedule=ScheduleKind(kind), lanes=97 if kind != "group-mapped" else 4 * gs,
                         group_size=gs, tiles_per_block=gs)
    _, pr, lanes = lwb.spmv_probe(dm, x, cfg)
    lib = _lib.load()
    code = {"thread-mapped": _lib.LW_THREAD_MAPPED, "merge-path": _lib.LW_MERGE_PATH,
            "group-mapped": _lib.LW_GROUP_MAPPED}[kind]
    need = lib.lw_spmv_workspace(code, m.rows, m.nnz, lanes, _lib.LW_F64)
    ws = torch.empty(max(need, 1), dtype=torch.uint8, device="cuda")
    y = torch.empty(m.rows, dtype=torch.float64, device="cuda")
    per_lane = torch.zeros(lanes, dtype=torch.int64, device="cuda")
    a_lane = torch.full((m.nnz,), -1, dtype=torch.int32, device="cuda")
    a_tile = torch.full((m.nnz,), -1, dtype=torch.int32, device="cuda")
    s = current_stream(dm.device)
    A = dm.c_struct()
    _lib.check(lib.lw_debug_lane_atom_counts(code, A, x.data_ptr(), y.data_ptr(), lanes, gs, gs,
                                             per_lane.data_ptr(), ws.data_ptr(), need, s), "debug counts")
    _lib.check(lib.lw_debug_atom_tiles(code, A, x.data_ptr(), y.data_ptr(), lanes, gs, gs, a_lane.data_ptr(),
                                       a_tile.data_ptr(), ws.data_ptr(), need, s), "debug tiles")
    np.testing.assert_array_equal(per_lane.cpu().numpy(), pr["lane_atoms"])
    np.testing.assert_array_equal(a_lane.cpu().numpy(), pr["atom_lane"])
    np.testing.assert_array_equal(a_tile.cpu().numpy(), pr["atom_tile"])
    rep = lwb.imbalance(lwb.csr_tile_set(m), dataclasses.replace(cfg, lanes=lanes))
    np.testing.assert_array_equal(per_lane.cpu().numpy(), rep.per_lane_atoms)
