"""Schedule sweep over the BASELINE.json configs (C1, C2b, C2u, C3, C4): every
schedule kernel, fp32 and fp64, with the reference CPU algorithm (oracle port,
all host threads) timed on the same matrix. One JSON line per measurement.

    python tools/bench_sweep.py [--configs C1,C2b,C2u,C3,C4] [--reps 20] [--out FILE]

GPU times: CUDA events around `reps` back-to-back launches after warm-up; for
matrices smaller than L2 (C1) a 512 MB buffer is written between reps and the
per-rep kernel time is taken from events around each launch (cold L2).
GB/s uses the SURVEY §8(d) byte model; frac is against MEASURED_PEAKS.json.
"""

from __future__ import annotations

import argparse
import json
import os
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
             ("group_warp", K.GROUP_MAPPED, 32), ("group_block", K.GROUP_MAPPED, 256)]


def peak():
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6650.0


def matrices(names):
    """Yield (config, label, DeviceCsr fp32, row stats)."""
    for name in names:
        if name == "C1":
            m = lwb.generate_random_csr(10_000, 10_000, 1_000_000, seed=1)
            yield "C1", "random 10k x 10k, 1M nnz, seed 1", m.to_device("float32"), m.row_offsets
        elif name == "C2b":
            d = lwb.generate_banded_device(1_000_000, 16, seed=2)
            yield "C2b", "banded 1M rows, half-bandwidth 16", d, d.row_offsets.cpu().numpy()
        elif name == "C2u":
            # device twin of generate_random_csr (the host generator takes minutes here)
            d = lwb.generate_uniform_device(1_000_000, 1_000_000, 32_000_000, seed=2)
            yield "C2u", "uniform 1M x 1M, 32M draws, seed 2 (device)", d, d.row_offsets.cpu().numpy()
        elif name == "C3":
            d = lwb.generate_rmat_csr(24, 16, seed=3)
            yield "C3", "R-MAT scale 24, ef 16, seed 3", d, d.row_offsets.cpu().numpy()
        elif name == "C4":
            for skew in (3.0, 2.0, 1.5, 1.2, 1.1, 1.05):
                m = lwb.generate_power_law_csr(1 << 20, 16.0, skew, seed=4)
                yield "C4", f"power-law 2^20 rows, avg 16, skew {skew}", m.to_device("float32"), m.row_offsets
            d = lwb.generate_uniform_device(1 << 20, 1 << 20, 16 << 20, seed=4)
            yield "C4", "uniform 2^20 x 2^20, 16 draws/row (device)", d, d.row_offsets.cpu().numpy()
            d = lwb.generate_banded_device(1 << 20, 8, seed=4)
            yield "C4", "banded 2^20 rows, half-bandwidth 8", d, d.row_offsets.cpu().numpy()


def time_gpu(A, x, cfg, reps, cold):
    y = lwb.spmv(A, x, cfg)
    for _ in range(3):
        lwb.spmv(A, x, cfg, out=y)
    torch.cuda.synchronize()
    if not cold:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            lwb.spmv(A, x, cfg, out=y)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps, y
    flush = torch.empty(128 << 20, dtype=torch.float32, device=A.device)   # 512 MB > L2
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lwb.spmv(A, x, cfg, out=y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), y


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2b,C2u,C3,C4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dtypes", default="float32,float64")
    ap.add_argument("--schedules", default="thread_mapped,work_oriented,group_warp,group_block")
    args = ap.parse_args()
    hbm = peak()
    threads = oracle.default_threads()
    out = open(args.out, "a") if args.out else None
    for cfgname, label, A32, off_host in matrices(args.configs.split(",")):
        stats = lwb.row_length_stats(off_host)
        for dtype in args.dtypes.split(","):
            A = A32 if dtype == "float32" else A32.astype("float64")
            x = torch.ones(A.cols, dtype=A.dtype, device=A.device)
            cold = A.algorithmic_bytes() < 256 << 20
            for sname, kind, gs in [s for s in SCHEDULES if s[0] in args.schedules.split(",")]:
                cfg = lwb.ExecutorConfig(schedule=kind, group_size=gs)
                ms, y = time_gpu(A, x, cfg, args.reps, cold)
                gbs = A.algorithmic_bytes() / (ms * 1e-3) / 1e9
                rec = {"config": cfgname, "matrix": label, "dtype": dtype, "schedule": sname,
                       "ms": round(ms, 4), "gflops": round(2 * A.nnz / (ms * 1e-3) / 1e9, 2),
                       "gbs": round(gbs, 1), "frac": round(gbs / hbm, 4), "l2": "cold" if cold else "streamed",
                       "rows": A.rows, "nnz": A.nnz, "row_stats": stats}
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
            del A
        if not args.no_cpu:
            off = A32.row_offsets.cpu().numpy().astype(np.int64)
            col = A32.col_indices.cpu().numpy().astype(np.int64)
            val = A32.values.cpu().numpy().astype(np.float64)
            xh = np.ones(A32.cols)
            for sname, kind in (("merge-path", "merge-path"), ("thread-mapped", "thread-mapped")):
                oracle.spmv(off, col, val, xh, kind, lanes=32 * threads, threads=threads)
                ts = []
                for _ in range(3):
                    t = time.perf_counter()
                    oracle.spmv(off, col, val, xh, kind, lanes=32 * threads, threads=threads)
                    ts.append(time.perf_counter() - t)
                sec = float(np.median(ts))
                rec = {"config": cfgname, "matrix": label, "dtype": "float64", "schedule": sname,
                       "impl": "cpu-reference-port", "cores": threads, "ms": round(sec * 1e3, 3),
                       "gflops": round(2 * A32.nnz / sec / 1e9, 3), "rows": A32.rows, "nnz": A32.nnz}
                line = json.dumps(rec)
                print(line, flush=True)
                if out:
                    out.write(line + "\n")
        del A32
        torch.cuda.empty_cache()
    if out:
        out.close()


if __name__ == "__main__":
    main()
