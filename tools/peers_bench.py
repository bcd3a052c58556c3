"""Time the fused-all-gather SpMV kernels (lw_spmv_work_oriented_peers[_hotx]) with P peer
buffers against the plain work_oriented SpMV on one GPU. Usage: python tools/peers_bench.py [scale] [P]"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402
from paper_2301_04792_b200 import _lib  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1
A = lw.generate_rmat_csr(scale, 16, seed=3)
x = torch.rand(A.cols, device="cuda")
y = torch.empty(A.rows, device="cuda")
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
bufs = [torch.empty(A.rows, device="cuda") for _ in range(P)]
ptrs = (ctypes.c_uint64 * P)(*[b.data_ptr() for b in bufs])
wo = lw.ExecutorConfig(schedule=lw.ScheduleKind.MERGE_PATH)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


need = lib.lw_spmv_work_oriented_workspace(A.rows, A.nnz, 0, _lib.LW_F32)
ws = torch.empty(need, dtype=torch.uint8, device="cuda")
print(f"plain   {timeit(lambda: lw.spmv(A, x, wo, out=y)):.4f} ms")
print(f"peers   {timeit(lambda: lib.lw_spmv_work_oriented_peers(A.c_struct(), x.data_ptr(), y.data_ptr(), 0, ws.data_ptr(), need, P, ptrs, 0, 0, st)):.4f} ms")
hx = A.pack_hot_columns()
need2 = lib.lw_spmv_work_oriented_hotx_workspace(A.rows, A.nnz, 0, hx.n_hot, _lib.LW_F32)
ws2 = torch.empty(need2, dtype=torch.uint8, device="cuda")
Hc = hx.packed.c_struct()
print(f"hot     {timeit(lambda: lw.spmv(A, x, wo, out=y)):.4f} ms")
print(f"hot+peers {timeit(lambda: lib.lw_spmv_work_oriented_peers_hotx(Hc, hx.hot_cols.data_ptr(), hx.n_hot, x.data_ptr(), y.data_ptr(), 0, ws2.data_ptr(), need2, P, ptrs, 0, 0, st)):.4f} ms")
