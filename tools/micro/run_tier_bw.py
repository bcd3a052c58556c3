"""Run tools/micro/tier_bw.cu on C3 (R-MAT 2^24, fp32): gather ceiling with a
shared-memory / DSMEM tier for the hottest x values.  Prints one JSON line per
configuration (time, Ggather/s, fraction of gathers served by the tier)."""
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
lib.tier_bw.restype = ctypes.c_int
lib.tier_max_clusters.restype = ctypes.c_int
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


def relabel(K):
    if K == 0:
        return col0, x[:1]
    slot = torch.full((A.cols,), -1, dtype=torch.int64, device="cuda")
    slot[order[:K]] = torch.arange(K, device="cuda")
    sl = slot[col0.long()]
    c = torch.where(sl >= 0, (sl | 0x80000000).to(torch.int64) - (1 << 32), col0.long()).to(torch.int32)
    return c, x[order[:K]].contiguous()


def run(mode, C, grid, nt, K, kloc, l1, reps=10):
    col, xh = relabel(K)
    smem = max(kloc * 4, 0)

    def f():
        rc = lib.tier_bw(mode, C, grid, nt, ctypes.c_long(smem), ctypes.c_void_p(col.data_ptr()),
                         ctypes.c_void_p(val.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                         ctypes.c_void_p(xh.data_ptr()), kloc, ctypes.c_void_p(out.data_ptr()),
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
    key = nt
    if key not in ref:
        ref[key] = o
    same = bool(torch.equal(o, ref[key]))
    cov = float(counts[order[:K]].sum()) / n if K else 0.0
    print(json.dumps({"mode": mode, "C": C, "grid": grid, "nt": nt, "K": K, "k_local": kloc, "l1": l1,
                      "ms": round(ms, 4), "Ggather_s": round(n / ms / 1e6, 1), "tier_frac": round(cov, 4),
                      "same_as_plain": same}), flush=True)


run(0, 1, SMS * 2, 1024, 0, 0, 1)
run(0, 1, SMS * 4, 512, 0, 0, 1)
run(0, 1, SMS, 1024, 0, 0, 1)
run(0, 1, SMS * 64, 1024, 0, 0, 1)
for K in (8192, 16384, 32768, 49152, 56320):
    for l1 in (1, 0):
        run(1, 1, SMS, 1024, K, K, l1)
for K in (8192, 16384, 27648):
    run(1, 1, SMS * 2, 512, K, K, 1)
for C in (2, 4, 8, 16):
    kloc = 49152
    mc = lib.tier_max_clusters(C, 1024, ctypes.c_long(kloc * 4))
    print(json.dumps({"C": C, "max_active_clusters": mc}), flush=True)
    if mc > 0:
        for l1 in (1, 0):
            run(2, C, mc * C, 1024, kloc * C, kloc, l1)
        mc2 = lib.tier_max_clusters(C, 512, ctypes.c_long(27648 * 4))
        if mc2 > 0:
            run(2, C, mc2 * C, 512, 27648 * C, 27648, 1)
