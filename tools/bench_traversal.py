"""SSSP / BFS throughput on an R-MAT graph (|hash weights|), every schedule, with the
reference CPU algorithm (C oracle port of lanework's frontier loop; the
reference's numba relax runs on one thread) timed on the same graph.

    python tools/bench_traversal.py [--scale 22] [--ef 16] [--reps 3] [--out F]

Metric: GTEPS = edges of the graph / traversal time (the usual Graph500-style
count; every pass is inside the timed region, including its host sync).
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
             ("group_warp", K.GROUP_MAPPED, 32), ("group_block", K.GROUP_MAPPED, 256)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=22)
    ap.add_argument("--ef", type=int, default=16)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    out = open(args.out, "a") if args.out else None

    def emit(rec):
        line = json.dumps(rec)
        print(line, flush=True)
        if out:
            out.write(line + "\n")

    A = lwb.generate_rmat_csr(args.scale, args.ef, seed=3, dtype="float64")
    G = lwb.DeviceCsr(A.rows, A.cols, A.row_offsets, A.col_indices, A.values.abs())
    off = G.row_offsets.cpu().numpy().astype(np.int64)
    src = int(np.argmax(np.diff(off)))
    label = f"rmat{args.scale}-ef{args.ef}-seed3 |w|"
    for op in ("sssp", "bfs"):
        fn = lwb.sssp if op == "sssp" else lwb.bfs
        for sname, kind, gs in SCHEDULES:
            cfg = lwb.ExecutorConfig(schedule=kind, group_size=gs)
            res, passes = fn(G, src, cfg, return_passes=True)
            torch.cuda.synchronize()
            ts = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn(G, src, cfg)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            reached = int((res < np.inf).sum().item()) if op == "sssp" else int((res >= 0).sum().item())
            emit({"op": op, "graph": label, "schedule": sname, "ms": round(ms, 3),
                  "gteps": round(G.nnz / (ms * 1e-3) / 1e9, 3), "passes": passes,
                  "vertices": G.rows, "edges": G.nnz, "reached": reached})
        if not args.no_cpu:
            col = G.col_indices.cpu().numpy().astype(np.int64)
            w = G.values.cpu().numpy()
            t = time.perf_counter()
            ref = oracle.sssp(off, col, w, src) if op == "sssp" else oracle.bfs(off, col, src)
            sec = time.perf_counter() - t
            same = bool(np.array_equal(ref, res.cpu().numpy()))
            emit({"op": op, "graph": label, "schedule": "frontier", "impl": "cpu-reference-port",
                  "cores": 1, "ms": round(sec * 1e3, 1), "gteps": round(G.nnz / sec / 1e9, 4),
                  "identical_to_gpu": same})
    if out:
        out.close()


if __name__ == "__main__":
    main()
