"""Ingestion throughput: Matrix Market text -> COO -> CSR with the native reader,
beside the reference's Python reader (when /root/reference is importable, i.e. in
the dev container only). One JSON line per measurement.

    python tools/bench_ingest.py [--entries 2000000] [--threads 0]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2301_04792_b200 as lw  # noqa: E402


def make_file(path, entries, rows, seed=5):
    rng = np.random.default_rng(seed)
    i = rng.integers(1, rows + 1, entries)
    j = rng.integers(1, rows + 1, entries)
    v = rng.normal(size=entries)
    with open(path, "w") as fh:
        fh.write(f"%%MatrixMarket matrix coordinate real general\n{rows} {rows} {entries}\n")
        fh.write("\n".join(f"{a} {b} {c!r}" for a, b, c in zip(i.tolist(), j.tolist(), v.tolist())))
        fh.write("\n")


def best(fn, reps=3):
    ts = []
    out = None
    for _ in range(reps):
        t = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t)
    return min(ts), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--entries", type=int, default=2_000_000)
    ap.add_argument("--rows", type=int, default=200_000)
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "m.mtx")
        make_file(path, args.entries, args.rows)
        mb = os.path.getsize(path) / 1e6
        t_parse, coo = best(lambda: lw.load_matrix_market(path, threads=args.threads))
        t_pack, csr = best(lambda: lw.coo_to_csr(coo, threads=args.threads))
        cores = len(os.sched_getaffinity(0))
        print(json.dumps({"impl": "native", "entries": args.entries, "file_mb": round(mb, 1),
                          "parse_s": round(t_parse, 4), "parse_mb_s": round(mb / t_parse, 1),
                          "coo_to_csr_s": round(t_pack, 4), "cores": cores}))
        ref = os.environ.get("LANEWORK_SRC", "/root/reference/pkg/src")
        if Path(ref).exists():
            sys.path.insert(0, ref)
            import lanework as ref_lw
            t_rp, rcoo = best(lambda: ref_lw.load_matrix_market(path), reps=1)
            t_rc, rcsr = best(lambda: ref_lw.coo_to_csr(rcoo), reps=1)
            same = (np.array_equal(rcsr.row_offsets, csr.row_offsets)
                    and np.array_equal(rcsr.col_indices, csr.col_indices)
                    and np.array_equal(rcsr.values, csr.values))
            print(json.dumps({"impl": "reference", "entries": args.entries, "file_mb": round(mb, 1),
                              "parse_s": round(t_rp, 4), "parse_mb_s": round(mb / t_rp, 1),
                              "coo_to_csr_s": round(t_rc, 4), "identical_csr": bool(same)}))


if __name__ == "__main__":
    main()
