"""Experiment: how much of the work_oriented time is the x gather? Same matrix,
columns remapped into a small (L1-resident) window vs the real columns."""
import sys
sys.path.insert(0, '.')
import torch
import paper_2301_04792_b200 as lwb

A = lwb.generate_rmat_csr(24, 16, 3)
cfg = lwb.ExecutorConfig(schedule=lwb.ScheduleKind.MERGE_PATH)
x = torch.ones(A.cols, device='cuda')


def t(M, reps=20):
    y = lwb.spmv(M, x, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lwb.spmv(M, x, cfg, out=y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("real cols      ms", t(A))
for mask in (0, 1023, 65535, (1 << 20) - 1):
    B = lwb.DeviceCsr(A.rows, A.cols, A.row_offsets, A.col_indices & mask, A.values)
    print(f"cols & {mask:8d} ms", t(B))
# columns made sequential per row (perfect spatial locality, same count)
seq = (torch.arange(A.nnz, device='cuda', dtype=torch.int64) % A.cols).to(torch.int32)
B = lwb.DeviceCsr(A.rows, A.cols, A.row_offsets, seq, A.values)
print("sequential cols ms", t(B))
