"""Reference point only (not a product path): cuSPARSE SpMV through
torch.sparse_csr_tensor @ x on the headline matrix, to place k_wo_chunk against
the vendor library on the same B200. Prints ms per SpMV for fp32 and fp64."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402

for dt in ("float32", "float64"):
    A = lw.generate_rmat_csr(24, 16, seed=3, dtype=dt)
    S = torch.sparse_csr_tensor(A.row_offsets, A.col_indices, A.values, size=(A.rows, A.cols))
    x = torch.ones(A.cols, 1, dtype=A.dtype, device="cuda")
    for _ in range(3):
        y = S @ x
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        y = S @ x
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    xo = torch.ones(A.cols, dtype=A.dtype, device="cuda")
    ours = lw.spmv(A, xo, lw.ExecutorConfig(schedule=lw.ScheduleKind.WORK_ORIENTED))
    ok = torch.allclose(ours.double(), y.double().squeeze(1), rtol=1e-4, atol=1e-3)
    print(f"cusparse {dt}: {ms:.3f} ms ({2 * A.nnz / ms / 1e6:.1f} GFLOP/s), agrees with ours: {ok}")
    del A, S, x, y
    torch.cuda.empty_cache()
