"""C5 operator layouts A/B (R-MAT 2^26 fp32, one GPU): per-SpMV time of the
work_oriented kernel on the matrix as generated, hot-x packed, degree-relabeled
(P A P^T), and relabeled + hot-x; one JSON line each (+ the one-time costs)."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2301_04792_b200 as lwb

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
A = lwb.generate_rmat_csr(scale, 16, seed=5)
cfg = lwb.ExecutorConfig(schedule=lwb.ScheduleKind.WORK_ORIENTED)
x = torch.rand(A.cols, device="cuda")
alg = A.algorithmic_bytes()


def t_spmv(M, v, reps=20):
    y = lwb.spmv(M, v, cfg)
    for _ in range(3):
        lwb.spmv(M, v, cfg, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lwb.spmv(M, v, cfg, out=y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, y


def emit(name, ms, **kw):
    print(json.dumps({"layout": name, "ms_per_spmv": round(ms, 4), "gbs": round(alg / ms / 1e6, 1),
                      **kw}), flush=True)


ms, y0 = t_spmv(A, x)
emit("plain", ms)
t = time.perf_counter(); A.pack_hot_columns(); torch.cuda.synchronize()
ms, y1 = t_spmv(A, x)
emit("hotx", ms, build_ms=round((time.perf_counter() - t) * 1e3, 1), same=bool(torch.equal(y0, y1)))
A.drop_hot_columns()
torch.cuda.synchronize()
t = time.perf_counter()
R = A.degree_relabel()
torch.cuda.synchronize()
build = (time.perf_counter() - t) * 1e3
xr = R.to_new(x)
ms, yr = t_spmv(R.matrix, xr)
back = R.to_old(yr)
err = float(((back.double() - y0.double()).abs().max()))
emit("relabel", ms, build_ms=round(build, 1), max_abs_diff_vs_plain=err)
t = time.perf_counter(); R.matrix.pack_hot_columns(); torch.cuda.synchronize()
ms, yr2 = t_spmv(R.matrix, xr)
emit("relabel+hotx", ms, build_ms=round((time.perf_counter() - t) * 1e3, 1), same=bool(torch.equal(yr, yr2)))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); R.to_old(yr); e1.record(); torch.cuda.synchronize()
print(json.dumps({"unpermute_ms": round(e0.elapsed_time(e1), 4)}))
