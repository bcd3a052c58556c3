"""Gather ceiling on C3 (R-MAT 2^24 fp32) when the columns are degree-relabeled
and the atoms of each G-atom group are sorted by column, laid out so that a
warp's gather instruction k reads 32 consecutive sorted columns (the layout a
'sorted-gather' SpMV would use).  Optionally the K hottest relabeled columns
are read from a shared-memory copy (tier_bw.cu mode 1)."""
import ctypes
import json
import subprocess
import sys

sys.path.insert(0, ".")
import torch

import paper_2301_04792_b200 as lwb

subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                "-o", "tools/micro/tier_bw.so", "tools/micro/tier_bw.cu"], check=True)
lib = ctypes.CDLL("tools/micro/tier_bw.so")
A = lwb.generate_rmat_csr(24, 16, 3)
SMS = torch.cuda.get_device_properties(0).multi_processor_count
n = (A.nnz // 16384) * 16384
col0 = A.col_indices[:n].contiguous().long()
val = A.values[:n].contiguous()
x = torch.rand(A.cols, device="cuda")
counts = torch.bincount(col0, minlength=A.cols)
order = torch.argsort(counts, descending=True)
rank = torch.empty(A.cols, dtype=torch.int64, device="cuda")
rank[order] = torch.arange(A.cols, device="cuda")
xr = x[order].contiguous()
out = torch.empty(n // 8 + 1024, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def layout(c, G):
    if G:
        c = torch.sort(c.view(-1, G), dim=1).values.reshape(-1)
        # warp block of 256 sorted columns: thread t's k-th atom = sorted element 32k + t
        c = c.view(-1, 8, 32).transpose(1, 2).reshape(-1)
    return c


def run(name, col, xx, mode=0, nt=512, K=0, reps=10):
    col = col.to(torch.int32).contiguous()
    if mode == 1:
        col = torch.where(col < K, col | (-0x80000000), col)
    grid = SMS * (2048 // nt) if mode == 0 else SMS
    xh = xx[:max(K, 1)].contiguous()

    def f():
        rc = lib.tier_bw(mode, 1, grid, nt, ctypes.c_long(K * 4), ctypes.c_void_p(col.data_ptr()),
                         ctypes.c_void_p(val.data_ptr()), ctypes.c_void_p(xx.data_ptr()),
                         ctypes.c_void_p(xh.data_ptr()), K, ctypes.c_void_p(out.data_ptr()),
                         ctypes.c_long(n), 1, ctypes.c_void_p(s))
        assert rc == 0, rc
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"name": name, "mode": mode, "nt": nt, "K": K, "ms": round(ms, 4),
                      "Ggather_s": round(n / ms / 1e6, 1)}), flush=True)


run("orig", col0, x)
run("relabel", rank[col0], xr)
for G in (256, 1024, 4096, 16384):
    run(f"orig sorted G={G}", layout(col0, G), x)
    rl = layout(rank[col0], G)
    run(f"relabel sorted G={G}", rl, xr)
    run(f"relabel sorted G={G} nt1024", rl, xr, nt=1024)
    run(f"relabel sorted G={G} + smem 32K", rl, xr, mode=1, nt=1024, K=32768)
    run(f"relabel sorted G={G} + smem 16K", rl, xr, mode=1, nt=1024, K=16384)
run("relabel + smem 32K", rank[col0], xr, mode=1, nt=1024, K=32768)
