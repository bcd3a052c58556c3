"""Experiment: hot-column packing of x (an inspector relabels columns so the most
gathered x values sit densely at the front of a packed x), unchanged kernel.
K hottest columns -> slots 0..K-1 of xp = [x[hot] | x]; other columns c -> K + c.
K = -1: full degree-sorted relabeling (xp = x[order]).
Prints the SpMV time per K, the pack (x -> xp) time, and bit-equality with the plain path."""
import sys, torch
sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
dt = torch.float64 if len(sys.argv) > 2 and sys.argv[2] == "f64" else torch.float32
Ks = [int(k) for k in sys.argv[3].split(",")] if len(sys.argv) > 3 else [2048, 4096, 8192, 16384, 32768, 65536, 131072, -1]
A = lw.generate_rmat_csr(scale, 16, seed=3, dtype="float64" if dt == torch.float64 else "float32")
x = torch.rand(A.cols, device="cuda", dtype=dt)
cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.WORK_ORIENTED)
ref = lw.spmv(A, x, cfg)
freq = torch.bincount(A.col_indices, minlength=A.cols)
order = torch.argsort(freq, descending=True, stable=True)


def timeit(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


y = torch.empty_like(ref)
print(f"plain {timeit(lambda: lw.spmv(A, x, cfg, out=y)):.4f} ms", flush=True)
for K in Ks:
    if K == -1:
        rank = torch.empty_like(order)
        rank[order] = torch.arange(A.cols, device="cuda")
        col = rank[A.col_indices.long()].to(torch.int32)
        idx = order
        xp = x[idx]
        ncols = A.cols
        pack = lambda: torch.index_select(x, 0, idx, out=xp)
    else:
        hot = order[:K]
        slot = torch.full((A.cols,), -1, dtype=torch.int64, device="cuda")
        slot[hot] = torch.arange(K, device="cuda")
        s = slot[A.col_indices.long()]
        col = torch.where(s >= 0, s, A.col_indices.long() + K).to(torch.int32)
        xp = torch.cat([x[hot], x])
        ncols = K + A.cols
        xh = xp[:K]
        pack = lambda: torch.index_select(x, 0, hot, out=xh)
    share = float(freq[order[: (A.cols if K == -1 else K)]].sum()) / A.nnz
    M = lw.DeviceCsr(A.rows, ncols, A.row_offsets, col, A.values)
    ms = timeit(lambda: lw.spmv(M, xp, cfg, out=y))
    pk = timeit(pack)
    print(f"K={K:7d} share {share:.3f}  spmv {ms:.4f} ms  pack {pk:.4f} ms  equal={torch.equal(y, ref)}", flush=True)
    del M, col
