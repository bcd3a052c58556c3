import sys, time, ctypes
sys.path.insert(0, '.')
import torch, numpy as np
import paper_2301_04792_b200 as lwb
from paper_2301_04792_b200 import _lib
lib = _lib.load()
A = lwb.generate_rmat_csr(int(sys.argv[1]) if len(sys.argv) > 1 else 22, 16, 3)
torch.cuda.synchronize()
h_off = A.row_offsets.cpu().pin_memory(); h_col = A.col_indices.cpu().pin_memory(); h_val = A.values.cpu().pin_memory()
h_x = torch.ones(A.cols).pin_memory(); h_y = torch.empty(A.rows).pin_memory()
print("pinned?", h_col.is_pinned(), h_val.is_pinned())
H = _lib.LwCsr(); H.rows, H.cols, H.nnz = A.rows, A.cols, A.nnz
H.row_offsets, H.col_indices, H.values = h_off.data_ptr(), h_col.data_ptr(), h_val.data_ptr()
H.offset_bits, H.dtype = 32, 0
s = torch.cuda.current_stream(); sp = int(s.cuda_stream)
for i in range(4):
    t = time.perf_counter(); rc = lib.lw_spmv_host(1, H, h_x.data_ptr(), h_y.data_ptr(), 0, 32, 32, sp); print("host call", rc, time.perf_counter() - t)
d = torch.empty(A.nnz, dtype=torch.int32, device='cuda')
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h_col, non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print("torch H2D col GB/s", A.nnz * 4 / dt / 1e9)
