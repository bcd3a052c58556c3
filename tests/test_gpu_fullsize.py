"""Parity at the sizes BASELINE.json names (C2b, C2u, C3, C4, C5), every schedule.

The oracle is lanework's merge-path SpMV (reference _fast.py:31-52 +
kernels.py:80-91, fp64 arithmetic — the reference's only precision,
kernels.py:60) restated in oracle/lw_oracle.c; `oracle.spmv_narrow` runs it
straight on the device layout copied back from the GPU (int32 columns,
fp32/fp64 values widened on load), with the reference CLI's lane count (32 x
host threads, cli.py:92), so a 1e9-atom matrix needs no 16 GB upcast. The gate
is the north star's per-entry bound |y - y_ref| <= rtol * sum_j |A_ij x_j|,
rtol 1e-5 (fp32) / 1e-12 (fp64), evaluated for every row.

Matrices:
  C2b  banded 1,000,000 rows, half-bandwidth 16           (32,999,728 atoms)
  C2u  uniform 1,000,000 x 1,000,000, 32M draws, seed 2   (device generator)
  C3   R-MAT scale 24, edge factor 16, seed 3             (263,430,552 atoms)
  C4   power-law 2^20 rows, mean 16, skews 3 .. 1.05, seed 4 (the reference's own
       generator), uniform 2^20 x 2^20 with 16 per row, banded 2^20 (hb 8)
  C5   R-MAT scale 26, edge factor 16, seed 5; 3 power iterations, each GPU
       iterate x_k fed to the oracle.
"""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2301_04792_b200 as lwb  # noqa: E402
from paper_2301_04792_b200 import ExecutorConfig, ScheduleKind  # noqa: E402

RTOL = {"float32": 1e-5, "float64": 1e-12}
K = ScheduleKind
# (id, kind, group_size, hot-x packed operands)
SCHEDULES = [("thread_mapped", K.THREAD_MAPPED, 32, False),
             ("work_oriented", K.WORK_ORIENTED, 32, False),
             ("work_oriented_hotx", K.WORK_ORIENTED, 32, True),
             ("group_warp", K.GROUP_MAPPED, 32, False),
             ("group_block", K.GROUP_MAPPED, 256, False)]
SCHED_IDS = [s[0] for s in SCHEDULES]


class Case:
    """One matrix in one value dtype: device operands, a seeded parity x (the
    reference CLI's x = rng(42).random(cols), cli.py:72) and the oracle's y, the
    latter computed once and shared by every schedule."""

    def __init__(self, build, dtype):
        self.A = build(dtype)
        g = np.random.default_rng(42).random(self.A.cols)
        self.x = torch.as_tensor(g).to("cuda", self.A.dtype)
        host = [t.cpu().numpy() for t in (self.A.row_offsets, self.A.col_indices, self.A.values)]
        self.y_ref, self.scale = oracle.spmv_narrow(*host, self.x.cpu().numpy())
        self.rtol = RTOL[dtype]

    def check(self, kind, gs, hot):
        A = self.A
        if hot:
            A.pack_hot_columns()
        try:
            y = lwb.spmv(A, self.x, ExecutorConfig(schedule=kind, group_size=gs))
        finally:
            if hot:
                A.drop_hot_columns()
        worst, row = oracle.worst_ratio(y.cpu().numpy(), self.y_ref, self.scale, self.rtol)
        assert worst <= 1.0, (f"row {row}: |y - y_ref| = {worst:.3g} x bound "
                              f"(y {float(y[row])}, ref {self.y_ref[row]})")
        return worst


_cache: dict = {}


def case(name, build, dtype):
    """Cached per matrix (both dtypes); one matrix resident at a time. The
    parametrisations below list the schedule outermost (it varies fastest) and
    the matrix innermost, so each matrix is built once."""
    if name not in _cache:
        _cache.clear()
        torch.cuda.empty_cache()
        _cache[name] = {}
    if dtype not in _cache[name]:
        _cache[name][dtype] = Case(build, dtype)
    return _cache[name][dtype]


def _c2b(dtype):
    return lwb.generate_banded_device(1_000_000, 16, seed=2, dtype=dtype)


def _c2u(dtype):
    return lwb.generate_uniform_device(1_000_000, 1_000_000, 32_000_000, seed=2, dtype=dtype)


def _c3(dtype):
    return lwb.generate_rmat_csr(24, 16, seed=3, dtype=dtype)


C4_SKEWS = [3.0, 2.0, 1.5, 1.2, 1.1, 1.05]
C4 = {f"powerlaw-skew{s}": (lambda dtype, s=s: lwb.generate_power_law_csr(1 << 20, 16.0, s, seed=4)
                            .to_device(dtype)) for s in C4_SKEWS}
C4["uniform"] = lambda dtype: lwb.generate_uniform_device(1 << 20, 1 << 20, 16 << 20, seed=4, dtype=dtype)
C4["banded"] = lambda dtype: lwb.generate_banded_device(1 << 20, 8, seed=4, dtype=dtype)


# ---- C2: 1M-row banded / uniform, group_mapped warp + block tiles and the rest ----------------

@pytest.mark.parametrize("sched", SCHEDULES, ids=SCHED_IDS)
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_c2b_banded_1m(sched, dtype):
    c = case("C2b", _c2b, dtype)
    assert c.A.rows == 1_000_000 and c.A.nnz == 32_999_728
    c.check(*sched[1:])


@pytest.mark.parametrize("sched", SCHEDULES, ids=SCHED_IDS)
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_c2u_uniform_1m(sched, dtype):
    c = case("C2u", _c2u, dtype)
    assert c.A.rows == 1_000_000 and 31_999_000 < c.A.nnz <= 32_000_000
    c.check(*sched[1:])


# ---- C3: the headline matrix, packed and unpacked work_oriented and every other kernel ----------

@pytest.mark.parametrize("sched", SCHEDULES, ids=SCHED_IDS)
@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_c3_rmat24(sched, dtype):
    c = case("C3", _c3, dtype)
    assert c.A.rows == 1 << 24 and c.A.nnz == 263_430_552
    c.check(*sched[1:])


def test_c3_hotx_packed_bit_identical_to_unpacked():
    """The packed headline kernel changes where x is read from, not the sums."""
    c = case("C3", _c3, "float32")
    cfg = ExecutorConfig(schedule=K.WORK_ORIENTED)
    y0 = lwb.spmv(c.A, c.x, cfg)
    c.A.pack_hot_columns()
    try:
        y1 = lwb.spmv(c.A, c.x, cfg)
    finally:
        c.A.drop_hot_columns()
    assert torch.equal(y0, y1)


# ---- C4: the row-length variance sweep, fp32 and fp64, every schedule ---------------------------

@pytest.mark.parametrize("sched", SCHEDULES, ids=SCHED_IDS)
@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("matrix", list(C4))
def test_c4_sweep(sched, matrix, dtype):
    c = case(f"C4-{matrix}", C4[matrix], dtype)
    assert c.A.rows == 1 << 20
    c.check(*sched[1:])


# ---- C5: 2^26-row R-MAT power iteration, every iterate checked ---------------------------------

@pytest.mark.parametrize("hot", [False, True], ids=["plain", "hotx"])
def test_c5_power_iteration_rmat26_per_iterate(hot):
    """x_{k+1} = A x_k / ||A x_k|| through distributed.power_iteration (world 1,
    the C5 driver), three iterations. Each GPU iterate x_k goes to the oracle,
    which computes y_ref = A x_k in fp64; the GPU's x_{k+1} must equal
    y_ref / ||y_ref|| within rtol * (sum_j |A_ij x_j| + |y_ref|) / ||y_ref|| — the
    SpMV bound plus the same relative bound on the norm."""
    from paper_2301_04792_b200.distributed import RowShard, nnz_balanced_bounds, power_iteration

    _cache.clear()
    torch.cuda.empty_cache()
    A = lwb.generate_rmat_csr(26, 16, seed=5, dtype="float32")
    assert A.rows == 1 << 26 and A.nnz > 1_000_000_000
    if hot:
        A.pack_hot_columns()
    host = [t.cpu().numpy() for t in (A.row_offsets, A.col_indices, A.values)]
    shard = RowShard(nnz_balanced_bounds(host[0], 1), 0)
    cfg = ExecutorConfig(schedule=K.WORK_ORIENTED)
    x = torch.full((A.rows,), 1.0 / np.sqrt(A.rows), dtype=torch.float32, device="cuda")
    for k in range(3):
        xk = x.cpu().numpy()
        x, norms = power_iteration(lambda v: lwb.spmv(A, v, cfg), A.rows, shard, 1, x0=x,
                                   dtype=torch.float32, device="cuda")
        y_ref, scale = oracle.spmv_narrow(*host, xk)
        nrm = float(np.linalg.norm(y_ref))
        assert abs(norms[-1] - nrm) <= 1e-5 * float(np.linalg.norm(scale)), (k, norms[-1], nrm)
        bound = 1e-5 * (scale + np.abs(y_ref)) / nrm
        err = np.abs(x.cpu().numpy().astype(np.float64) - y_ref / nrm)
        worst = float((err / np.maximum(bound, 1e-300)).max())
        assert worst <= 1.0, f"iterate {k + 1}: worst err/bound {worst:.3g}"
    del A
    torch.cuda.empty_cache()


def test_c5_relabeled_inplace_driver_per_iterate():
    """The bench's C5 path: degree-relabeled operator P A P^T (+ hot-x), the
    in-place gather-layout driver, iterates mapped back to the original
    numbering and checked against the oracle on the ORIGINAL matrix."""
    from paper_2301_04792_b200.distributed import GatherLayout, power_iteration_inplace

    _cache.clear()
    torch.cuda.empty_cache()
    A = lwb.generate_rmat_csr(26, 16, seed=5, dtype="float32")
    host = [t.cpu().numpy() for t in (A.row_offsets, A.col_indices, A.values)]
    R = A.degree_relabel()
    n = A.rows
    del A
    lay = GatherLayout(np.array([0, n]), 1)
    M = lay.remap_columns(R.matrix)
    M.pack_hot_columns()
    cfg = ExecutorConfig(schedule=K.WORK_ORIENTED)

    def local(x, r0, r1, out):
        lwb.spmv(M, x, cfg, out=out)

    x = torch.full((n,), 1.0 / np.sqrt(n), dtype=torch.float32, device="cuda")
    for k in range(3):
        xk = x.cpu().numpy()
        xb, norms = power_iteration_inplace(local, lay, 1, x0=lay.to_layout(R.to_new(x)),
                                            dtype=torch.float32, device="cuda")
        x = R.to_old(lay.from_layout(xb))
        y_ref, scale = oracle.spmv_narrow(*host, xk)
        nrm = float(np.linalg.norm(y_ref))
        assert abs(norms[-1] - nrm) <= 1e-5 * float(np.linalg.norm(scale)), (k, norms[-1], nrm)
        bound = 1e-5 * (scale + np.abs(y_ref)) / nrm
        err = np.abs(x.cpu().numpy().astype(np.float64) - y_ref / nrm)
        worst = float((err / np.maximum(bound, 1e-300)).max())
        assert worst <= 1.0, f"iterate {k + 1}: worst err/bound {worst:.3g}"


def test_degree_relabel_keeps_row_sums():
    """P A P^T: row i' of the relabeled matrix is row order[i'] with renamed
    columns and the atoms in their original order, so y' = P y bit for bit
    (integer data: exact in any summation order, so bit-equal)."""
    A = lwb.generate_rmat_csr(18, 16, seed=2, dtype="float64")
    A.values.copy_(torch.randint(-4, 5, (A.nnz,), device="cuda").to(torch.float64))   # exact sums
    R = A.degree_relabel()
    x = torch.randint(-3, 4, (A.cols,), device="cuda").to(torch.float64)
    tm = ExecutorConfig(schedule=K.THREAD_MAPPED)
    y = lwb.spmv(A, x, tm)
    yr = lwb.spmv(R.matrix, R.to_new(x), tm)
    assert torch.equal(R.to_old(yr), y)
    counts = torch.bincount(R.matrix.col_indices.long(), minlength=A.cols)
    assert bool((counts[:-1] >= counts[1:]).all())   # columns by decreasing degree
