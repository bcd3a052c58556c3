import sys, torch
sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw
A = lw.generate_rmat_csr(24, 16, seed=3)
U = lw.DeviceCsr(A.rows, A.cols, A.row_offsets, torch.randint(0, A.cols, (A.nnz,), device="cuda", dtype=torch.int32), A.values)
for M in (A, U):
    for _ in range(2):
        M.drop_hot_columns(); M.pack_hot_columns()
torch.cuda.synchronize()
