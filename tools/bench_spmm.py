"""SpMM sweep (C = A B, B dense [cols, n] row-major), fp32, every schedule, with the
reference CPU algorithm (C oracle port of lanework.spmm, all host threads) timed on
a bounded row sample of the same matrix. One JSON line per measurement.

    python tools/bench_spmm.py [--configs C2u,C2b,C3] [--ns 4,16,64] [--reps 10] [--out F]

Byte model per SpMM: nnz*(4 + s) + (rows+1)*4 + cols*n*s (B read
once) + rows*n*s (C written); FLOPs 2*nnz*n. Matrices are far larger than L2.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2301_04792_b200 as lwb  # noqa: E402
from oracle import oracle  # noqa: E402

K = lwb.ScheduleKind
SCHEDULES = [("thread_mapped", K.THREAD_MAPPED, 32), ("work_oriented", K.MERGE_PATH, 32),
             ("group_warp", K.GROUP_MAPPED, 32)]


def peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0


def matrix(name):
    if name == "C2u":
        return "random 1M x 1M, 32M nnz, seed 2", lwb.generate_random_csr(
            1_000_000, 1_000_000, 32_000_000, seed=2).to_device("float32")
    if name == "C2b":
        return "banded 1M rows, half-bandwidth 16", lwb.generate_banded_device(1_000_000, 16, seed=2)
    if name == "C3":
        return "R-MAT scale 24, ef 16, seed 3", lwb.generate_rmat_csr(24, 16, seed=3)
    if name == "C3s":
        return "R-MAT scale 22, ef 16, seed 3", lwb.generate_rmat_csr(22, 16, seed=3)
    raise ValueError(name)


def spmm_bytes(A, n):
    s = A.values.element_size()
    return A.nnz * (4 + s) + (A.rows + 1) * A.row_offsets.element_size() + A.cols * n * s + A.rows * n * s


def time_gpu(A, B, cfg, reps):
    C = lwb.spmm(A, B, cfg)
    for _ in range(2):
        lwb.spmm(A, B, cfg, out=C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lwb.spmm(A, B, cfg, out=C)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def cpu_sample(A, n, threads, target_nnz=4_000_000):
    """Reference SpMM (oracle port, merge-path, 32 lanes per thread) on a row sample."""
    off = A.row_offsets.cpu().numpy().astype(np.int64)
    stop = int(np.searchsorted(off, min(target_nnz, A.nnz), side="left"))
    stop = max(1, min(stop, A.rows))
    offs = off[:stop + 1]
    nnz = int(offs[-1])
    col = A.col_indices[:nnz].cpu().numpy().astype(np.int64)
    val = A.values[:nnz].cpu().numpy().astype(np.float64)
    B = np.ones((A.cols, n))
    oracle.spmm(offs, col, val, B, "merge-path", lanes=32 * threads, threads=threads)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        oracle.spmm(offs, col, val, B, "merge-path", lanes=32 * threads, threads=threads)
        ts.append(time.perf_counter() - t)
    sec = float(np.median(ts))
    return 2.0 * nnz * n / sec / 1e9, sec, stop, nnz


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2u,C2b,C3")
    ap.add_argument("--ns", default="4,16,64")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--schedules", default="thread_mapped,work_oriented,group_warp")
    args = ap.parse_args()
    hbm = peak()
    threads = oracle.default_threads()
    want = set(args.schedules.split(","))
    out = open(args.out, "a") if args.out else None

    def emit(rec):
        line = json.dumps(rec)
        print(line, flush=True)
        if out:
            out.write(line + "\n")

    for name in args.configs.split(","):
        label, A = matrix(name)
        for n in [int(v) for v in args.ns.split(",")]:
            B = torch.ones((A.cols, n), dtype=A.dtype, device=A.device)
            nb = spmm_bytes(A, n)
            for sname, kind, gs in SCHEDULES:
                if sname not in want:
                    continue
                ms = time_gpu(A, B, lwb.ExecutorConfig(schedule=kind, group_size=gs), args.reps)
                gbs = nb / (ms * 1e-3) / 1e9
                emit({"op": "spmm", "config": name, "matrix": label, "n": n, "dtype": "float32",
                      "schedule": sname, "ms": round(ms, 4),
                      "gflops": round(2 * A.nnz * n / (ms * 1e-3) / 1e9, 2),
                      "gbs": round(gbs, 1), "frac": round(gbs / hbm, 4), "alg_bytes": nb,
                      "rows": A.rows, "nnz": A.nnz})
            if not args.no_cpu:
                gf, sec, rows_s, nnz_s = cpu_sample(A, n, threads)
                emit({"op": "spmm", "config": name, "matrix": label, "n": n, "dtype": "float64",
                      "schedule": "merge-path", "impl": "cpu-reference-port", "cores": threads,
                      "gflops": round(gf, 3), "sample": f"first {rows_s} rows ({nnz_s} nnz)",
                      "ms_sample": round(sec * 1e3, 3)})
            del B
        del A
        torch.cuda.empty_cache()
    if out:
        out.close()


if __name__ == "__main__":
    main()
