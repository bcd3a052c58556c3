"""Projected strong scaling from per-shard measurements on ONE B200 (the sandbox
grants one GPU; `bench.py --gpus N` is the real N-GPU run).

For G in 1, 2, 4, 8: the matrix is cut with distributed.row_bounds — nnz-
balanced (the north star's split) and rows+nnz-balanced (the work_oriented
partition across GPUs, bench.py's default) — every shard is copied out and hot-x packed
like a rank's operator, and its full SpMV step (partition + chunk + fix-up) is
timed on cuda:0 with CUDA events. Since a single SpMV shards with no exchange
(x replicated), G GPUs would finish in max_g t_g: the projected
aggregate is 2·nnz / max_g t_g. C5 adds the per-iteration all-gather volume
((G-1)/G · rows · 4 B received per GPU) and its time at 900 GB/s as an ESTIMATE
(not measured here). One JSON line per (workload, G).

    python tools/shard_projection.py [--c5]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402
from paper_2301_04792_b200.distributed import row_bounds  # noqa: E402


def step_ms(A, reps=20):
    x = torch.ones(A.cols, device="cuda", dtype=A.dtype)
    y = torch.empty(A.rows, device="cuda", dtype=A.dtype)
    cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.WORK_ORIENTED)
    for _ in range(5):
        lw.spmv(A, x, cfg, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lw.spmv(A, x, cfg, out=y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(name, full, relabel=False, balance="work"):
    if relabel:
        full = full.degree_relabel().matrix
    nnz, rows = full.nnz, full.rows
    off = full.row_offsets.cpu().numpy()
    base = None
    for G in (1, 2, 4, 8):
        b = row_bounds(off, G, balance)
        ts, shard_nnz, shard_rows = [], [], []
        for g in range(G):
            S = full.row_slice(int(b[g]), int(b[g + 1]))
            S = lw.DeviceCsr(S.rows, S.cols, S.row_offsets.clone(), S.col_indices.clone(), S.values.clone())
            S.pack_hot_columns()
            ts.append(step_ms(S))
            shard_nnz.append(S.nnz)
            shard_rows.append(S.rows)
            del S
            torch.cuda.empty_cache()
        tmax = max(ts)
        base = base or tmax
        line = {"workload": name, "balance": balance, "G": G, "shard_ms": [round(t, 4) for t in ts],
                "shard_nnz": shard_nnz, "shard_rows": shard_rows, "max_ms": round(tmax, 4),
                "projected_gflops": round(2.0 * nnz / (tmax * 1e-3) / 1e9, 1),
                "projected_speedup": round(base / tmax, 2), "projected_efficiency": round(base / tmax / G, 3),
                "source": "per-shard SpMV steps timed one after another on one B200 (projection, not an N-GPU run)"}
        if name.startswith("rmat26"):
            recv = (G - 1) / G * rows * 4
            line["allgather_mb_per_gpu"] = round(recv / 1e6, 1)
            line["allgather_ms_at_900GBps_estimate"] = round(recv / 900e9 * 1e3, 3)
        print(json.dumps(line), flush=True)


def main():
    A = lw.generate_rmat_csr(24, 16, seed=3)
    bals = sys.argv[sys.argv.index("--balances") + 1].split(",") if "--balances" in sys.argv else ["nnz", "work"]
    for bal in bals:
        run("rmat24-ef16-seed3 (C3)", A, balance=bal)
    del A
    if "--c5" in sys.argv:
        A = lw.generate_rmat_csr(26, 16, seed=5).degree_relabel().matrix
        for bal in bals:
            run("rmat26-ef16-seed5 (C5 operator, relabeled)", A, balance=bal)


if __name__ == "__main__":
    main()
