import sys, torch
sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw
from paper_2301_04792_b200.distributed import row_bounds
A = lw.generate_rmat_csr(24, 16, seed=3)
b = row_bounds(A.row_offsets.cpu().numpy(), 8)
S = A.row_slice(int(b[7]), int(b[8]))
S = lw.DeviceCsr(S.rows, S.cols, S.row_offsets.clone(), S.col_indices.clone(), S.values.clone())
S.pack_hot_columns()
x = torch.ones(S.cols, device="cuda"); y = torch.empty(S.rows, device="cuda")
cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.WORK_ORIENTED)
for _ in range(8): lw.spmv(S, x, cfg, out=y)
torch.cuda.synchronize()
print("rows", S.rows, "nnz", S.nnz)
