"""Gather ceiling on C3 (R-MAT 2^24 fp32) when the K most gathered columns are
relabeled to a dense prefix of x (x2 = [x[hot] | x], hot gathers read the
prefix): does a larger dense hot region keep more gathers in L1?"""
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
n = (A.nnz // 8192) * 8192
col0 = A.col_indices[:n].contiguous()
val = A.values[:n].contiguous()
x = torch.rand(A.cols, device="cuda")
counts = torch.bincount(col0.long(), minlength=A.cols)
order = torch.argsort(counts, descending=True)
out = torch.empty(n // 8 + 1024, device="cuda")
s = torch.cuda.current_stream().cuda_stream
ref = {}
full_perm = None


def relabel(K, full):
    """hot -> slot in [0, K); cold -> K + original column (x2 = [x[hot] | x]).
    full: a complete degree-ordered relabeling (x2 = x[order])."""
    if full:
        rank = torch.empty(A.cols, dtype=torch.int64, device="cuda")
        rank[order] = torch.arange(A.cols, device="cuda")
        return rank[col0.long()].to(torch.int32), x[order].contiguous()
    slot = torch.full((A.cols,), -1, dtype=torch.int64, device="cuda")
    slot[order[:K]] = torch.arange(K, device="cuda")
    sl = slot[col0.long()]
    c = torch.where(sl >= 0, sl, col0.long() + K).to(torch.int32)
    return c, torch.cat([x[order[:K]], x]).contiguous()


def run(mode, K, l1, full=False, nt=512, reps=10):
    col, x2 = relabel(K, full)
    grid = SMS * (2048 // nt)

    def f():
        rc = lib.tier_bw(mode, 1, grid, nt, ctypes.c_long(0), ctypes.c_void_p(col.data_ptr()),
                         ctypes.c_void_p(val.data_ptr()), ctypes.c_void_p(x2.data_ptr()),
                         ctypes.c_void_p(x2.data_ptr()), K, ctypes.c_void_p(out.data_ptr()),
                         ctypes.c_long(n), l1, ctypes.c_void_p(s))
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
    o = out[: n // 8].clone()
    if nt not in ref:
        ref[nt] = o
    cov = float(counts[order[:K]].sum()) / n if K else 0.0
    print(json.dumps({"mode": mode, "K": K, "full": full, "l1": l1, "nt": nt, "ms": round(ms, 4),
                      "Ggather_s": round(n / ms / 1e6, 1), "hot_frac": round(cov, 4),
                      "same": bool(torch.equal(o, ref[nt]))}), flush=True)


run(0, 0, 1)
for K in (12288, 49152, 196608, 1 << 20, 1 << 22):
    run(0, K, 1)
    run(3, K, 1)
run(0, A.cols, 1, full=True)
run(0, A.cols, 1, full=True, nt=1024)
