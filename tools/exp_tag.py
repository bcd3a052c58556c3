"""Experiment: hot-column tagging (bit 31 of col) with L1 evict_last for hot columns and
L1::no_allocate for the rest. Needs the LW_EXP_TAG build (LWB200_LIB=variants/tag.so)."""
import os, sys, torch
sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw
A = lw.generate_rmat_csr(24, 16, seed=3)
x = torch.rand(A.cols, device="cuda")
cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.WORK_ORIENTED)
ref = lw.spmv(A, x, cfg)
freq = torch.bincount(A.col_indices, minlength=A.cols)
order = torch.argsort(freq, descending=True)
def timeit(M):
    y = torch.empty_like(ref)
    for _ in range(3): lw.spmv(M, x, cfg, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): lw.spmv(M, x, cfg, out=y)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 20, y
line_freq = torch.zeros((A.cols + 31) // 32, dtype=torch.int64, device="cuda")
line_freq.index_add_(0, torch.arange(A.cols, device="cuda") // 32, freq)
lorder = torch.argsort(line_freq, descending=True)
for L in [0, 256, 512, 768, 1024, 1536, 2048]:
    hot_line = torch.zeros(line_freq.numel(), dtype=torch.bool, device="cuda")
    if L: hot_line[lorder[:L]] = True
    hot = hot_line[torch.arange(A.cols, device="cuda") // 32]
    covered = float(line_freq[lorder[:L]].sum()) / A.nnz if L else 0.0
    col = A.col_indices | (hot[A.col_indices.long()].int() << 31)
    M = lw.DeviceCsr(A.rows, A.cols, A.row_offsets, col.to(torch.int32), A.values)
    ms, y = timeit(M)
    print(f"lines={L:5d} ({L * 128 // 1024} KB) hot share {covered:.3f}  {ms:.4f} ms  equal={torch.equal(y, ref)}", flush=True)
