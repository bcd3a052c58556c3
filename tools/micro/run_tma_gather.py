"""Run tools/micro/tma_gather.cu on C3's column stream (R-MAT 2^24, fp32): gather
throughput when NTMA of each thread's 8 gathers go through TMA gather4 instead of
the LSU. Prints one JSON line per configuration; checks every sum against NTMA=0."""
import ctypes
import json
import subprocess
import sys

sys.path.insert(0, ".")
import torch

import paper_2301_04792_b200 as lwb

subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                "-o", "tools/micro/tma_gather.so", "tools/micro/tma_gather.cu"], check=True)
lib = ctypes.CDLL("tools/micro/tma_gather.so")
A = lwb.generate_rmat_csr(24, 16, 3)
n = (A.nnz // 8192) * 8192
col = A.col_indices[:n].contiguous()
val = A.values[:n].contiguous()
x = torch.rand(A.cols, device="cuda")
out = torch.empty(n // 8, device="cuda")
s = torch.cuda.current_stream().cuda_stream
ref = {}
ucol = torch.randint(0, A.cols, (n,), device="cuda", dtype=torch.int32)


def run(nt, ntma, c, tag, reps=10):
    def f():
        rc = lib.tma_gather(nt, ntma, ctypes.c_void_p(c.data_ptr()), ctypes.c_void_p(val.data_ptr()),
                            ctypes.c_void_p(x.data_ptr()), ctypes.c_long(A.cols), ctypes.c_void_p(out.data_ptr()),
                            ctypes.c_long(n), ctypes.c_void_p(s))
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
    key = (tag, nt)
    o = out.clone()
    if ntma == 0:
        ref[key] = o
    same = bool(torch.allclose(o, ref[key], rtol=1e-5, atol=1e-5)) if key in ref and ntma >= 0 else None
    print(json.dumps({"cols": tag, "nt": nt, "ntma": ntma, "ms": round(ms, 4),
                      "Ggather_s": round(n / ms / 1e6, 1), "same_as_lsu": same}), flush=True)


if len(sys.argv) > 1 and sys.argv[1] == "tr":
    for tag, c in (("c3", col), ("uniform", ucol)):
        run(512, 0, c, tag)
        run(512, -1, c, tag)
    sys.exit(0)
for tag, c in (("c3", col), ("uniform", ucol)):
    for nt in (512, 256):
        for ntma in (0, 4, 8):
            run(nt, ntma, c, tag)
    run(128, 4, c, tag)
    run(128, 8, c, tag)
