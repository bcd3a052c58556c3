"""Hot-x packing through the library API: build time, SpMV time plain vs packed
(max_hot sweep), bit-equality. Usage: python tools/hotx_bench.py [scale] [f32|f64] [K,K,...]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dt = "float64" if len(sys.argv) > 2 and sys.argv[2] == "f64" else "float32"
Ks = [int(k) for k in sys.argv[3].split(",")] if len(sys.argv) > 3 else [None]
A = lw.generate_rmat_csr(scale, 16, seed=3, dtype=dt)
x = torch.rand(A.cols, device="cuda", dtype=A.dtype)
cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.WORK_ORIENTED)
y = lw.spmv(A, x, cfg)
ref = y.clone()


def timeit(n=30):
    for _ in range(5):
        lw.spmv(A, x, cfg, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        lw.spmv(A, x, cfg, out=y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


print(f"scale {scale} {dt} nnz {A.nnz}: plain {timeit():.4f} ms", flush=True)
for K in Ks:
    A.drop_hot_columns()
    torch.cuda.synchronize()
    t = time.perf_counter()
    hx = A.pack_hot_columns(K)
    torch.cuda.synchronize()
    bt = (time.perf_counter() - t) * 1e3
    ms = timeit()
    print(f"max_hot {hx.max_hot:6d} n_hot {hx.n_hot:6d} build {bt:8.1f} ms  spmv {ms:.4f} ms  "
          f"equal={torch.equal(y, ref)}", flush=True)

if "--freq-order" in sys.argv:
    # same hot set, slots in descending gather count instead of ascending column
    from paper_2301_04792_b200.device import DeviceCsr, HotColumns
    counts = torch.bincount(A.col_indices, minlength=A.cols)
    for K in Ks:
        A.drop_hot_columns()
        hx = A.pack_hot_columns(K)
        o = torch.argsort(counts[hx.hot_cols.long()], descending=True, stable=True)
        hot = hx.hot_cols[o].contiguous()
        slot = torch.full((A.cols,), -1, dtype=torch.int64, device="cuda")
        slot[hot.long()] = torch.arange(hx.n_hot, device="cuda")
        s = slot[A.col_indices.long()]
        col = torch.where(s >= 0, s | (1 << 31), A.col_indices.long()).to(torch.int64)
        col = (col & 0xFFFFFFFF).to(torch.uint32).view(torch.int32) if hasattr(torch, "uint32") else col.int()
        packed = DeviceCsr(A.rows, A.cols, A.row_offsets, col.contiguous(), A.values)
        A.__dict__["_hotx"] = HotColumns(packed, hot, hx.n_hot, hx.max_hot, hx.key)
        ms = timeit()
        print(f"freq-order max_hot {hx.max_hot:6d} spmv {ms:.4f} ms equal={torch.equal(y, ref)}", flush=True)
