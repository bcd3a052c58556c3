import ctypes, sys
sys.path.insert(0, '.')
import torch
import paper_2301_04792_b200 as lwb
lib = ctypes.CDLL('tools/micro/gather_bw.so')
A = lwb.generate_rmat_csr(24, 16, 3)
n = (A.nnz // 32) * 32
x = torch.rand(A.cols, device='cuda')
out = torch.empty(n // 8 + 1, device='cuda')
s = torch.cuda.current_stream().cuda_stream
def t(mode, col):
    f = lambda: lib.gather_bw(mode, ctypes.c_void_p(col.data_ptr()), ctypes.c_void_p(A.values.data_ptr()),
                              ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), ctypes.c_long(n), ctypes.c_void_p(s))
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10
for name, mode, col in [("ipt16 gather rmat", 0, A.col_indices), ("ipt16 no-gather", 1, A.col_indices),
                        ("ipt8 gather rmat", 2, A.col_indices), ("ipt32 gather rmat", 3, A.col_indices),
                        ("ipt16 gather cols&0", 0, A.col_indices & 0),
                        ("ipt16 gather uniform", 0, torch.randint(0, A.cols, (A.nnz,), device='cuda', dtype=torch.int32))]:
    ms = t(mode, col)
    print(f"{name:24s} {ms:.3f} ms   stream {n * 8 / ms / 1e6:.0f} GB/s  {n / ms / 1e6:.0f} Ggather/s")
