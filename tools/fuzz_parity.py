"""Randomised parity sweep (not part of the test suite): random CSR shapes and row-length
mixes (empty runs, single huge rows, power-law), every schedule and group shape, explicit
and auto lane counts, fp32 / fp64, int32 / int64 offsets, hot-x packed and not — each y
against the C oracle with the north star's bound (integer data: bit-exact).

    python tools/fuzz_parity.py [seconds] [seed]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402
from oracle import oracle  # noqa: E402

K = lw.ScheduleKind


def random_csr(rng):
    rows = int(rng.integers(1, 40_000))
    cols = int(rng.integers(1, 50_000))
    mode = rng.integers(0, 4)
    if mode == 0:
        lengths = rng.integers(0, 40, size=rows)
    elif mode == 1:
        lengths = np.minimum((rng.zipf(1.3, rows) - 1), cols)
    elif mode == 2:
        lengths = rng.integers(0, 3, size=rows)
        lengths[rng.integers(0, rows)] = min(cols, int(rng.integers(1000, 200_000)))
    else:
        lengths = rng.integers(0, 10, size=rows)
        a = int(rng.integers(0, rows))
        lengths[a:a + int(rng.integers(0, 20_000))] = 0
    lengths = np.minimum(lengths, cols)
    off = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    col = np.concatenate([np.sort(rng.choice(cols, size=int(n), replace=False)) for n in lengths if n]
                         or [np.zeros(0, np.int64)]).astype(np.int64)
    integer = bool(rng.integers(0, 2))
    val = (rng.integers(-3, 4, size=col.size).astype(np.float64) if integer
           else rng.random(col.size) * 2 - 1)
    x = rng.integers(-3, 4, size=cols).astype(np.float64) if integer else rng.random(cols)
    return off, col, val, x, rows, cols, integer


def spmm_sweep(budget, rng):
    """The same for SpMM (n = 1..70 columns of B) under every schedule."""
    t_end = time.time() + budget
    n_cases = n_runs = 0
    while time.time() < t_end:
        off, col, val, x, rows, cols, integer = random_csr(rng)
        n = int(rng.integers(1, 70))
        B = (rng.integers(-3, 4, size=(cols, n)).astype(np.float64) if integer else rng.random((cols, n)))
        want = oracle.spmm(off, col, val, B, "thread-mapped", lanes=1)
        scale = oracle.abs_spmm_sums(off, col, val, B)
        for dt in (torch.float32, torch.float64):
            if not integer and dt == torch.float32:
                continue   # fp32 rounding of B/values: covered by the SpMV sweep's fp32 path
            m = lw.DeviceCsr(rows, cols, torch.as_tensor(off).cuda().to(torch.int32),
                             torch.as_tensor(col).cuda().to(torch.int32), torch.as_tensor(val).cuda().to(dt))
            Bt = torch.as_tensor(B).cuda().to(dt)
            for cfg in (lw.ExecutorConfig(schedule=K.THREAD_MAPPED), lw.ExecutorConfig(schedule=K.MERGE_PATH),
                        lw.ExecutorConfig(schedule=K.GROUP_MAPPED, group_size=32),
                        lw.ExecutorConfig(schedule=K.GROUP_MAPPED, lanes=int(rng.integers(1, 3000)),
                                          group_size=int(rng.integers(1, 300)),
                                          tiles_per_block=int(rng.integers(1, 300)))):
                C = lw.spmm(m, Bt, cfg).double().cpu().numpy()
                ok = np.array_equal(C, want) if integer else oracle.tolerance_ok(C, want, scale, 1e-12)[0]
                n_runs += 1
                if not ok:
                    print("SPMM MISMATCH", dict(rows=rows, cols=cols, n=n, dtype=str(dt), cfg=str(cfg)), flush=True)
                    return 1
        n_cases += 1
    print(f"spmm fuzz ok: {n_cases} matrices, {n_runs} SpMMs", flush=True)
    return 0


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    if "--spmm" in sys.argv:
        return spmm_sweep(budget, rng)
    t_end = time.time() + budget
    n_cases = n_runs = 0
    while time.time() < t_end:
        off, col, val, x, rows, cols, integer = random_csr(rng)
        want = oracle.spmv(off, col, val, x, "merge-path", lanes=64)
        scale = oracle.abs_row_sums(off, col, val, x)
        for dt in (torch.float32, torch.float64):
            if not integer and dt == torch.float32:
                v32 = val.astype(np.float32).astype(np.float64)
                x32 = x.astype(np.float32).astype(np.float64)
                want_d = oracle.spmv(off, col, v32, x32, "merge-path", lanes=64)
                scale_d = oracle.abs_row_sums(off, col, v32, x32)
            else:
                want_d, scale_d = want, scale
            bits = int(rng.choice([32, 64]))
            odt = torch.int32 if bits == 32 else torch.int64
            m = lw.DeviceCsr(rows, cols, torch.as_tensor(off).cuda().to(odt), torch.as_tensor(col).cuda().to(torch.int32),
                             torch.as_tensor(val).cuda().to(dt))
            xt = torch.as_tensor(x).cuda().to(dt)
            cfgs = [lw.ExecutorConfig(schedule=K.THREAD_MAPPED), lw.ExecutorConfig(schedule=K.MERGE_PATH),
                    lw.ExecutorConfig(schedule=K.GROUP_MAPPED, group_size=32),
                    lw.ExecutorConfig(schedule=K.GROUP_MAPPED, group_size=256),
                    lw.ExecutorConfig(schedule=K.GROUP_MAPPED, lanes=int(rng.integers(1, 3000)),
                                      group_size=int(rng.integers(1, 300)), tiles_per_block=int(rng.integers(1, 300))),
                    lw.ExecutorConfig(schedule=K.MERGE_PATH, lanes=int(rng.integers(1, 5000)))]
            for pack in (False, True):
                if pack:
                    m.pack_hot_columns(int(rng.integers(1, 20000)))
                for cfg in cfgs:
                    y = lw.spmv(m, xt, cfg).double().cpu().numpy()
                    if integer:
                        ok = np.array_equal(y, want_d)
                        worst = float(np.abs(y - want_d).max()) if y.size else 0.0
                    else:
                        ok, worst = oracle.tolerance_ok(y, want_d, scale_d, 1e-5 if dt == torch.float32 else 1e-12)
                    n_runs += 1
                    if not ok:
                        print("MISMATCH", dict(rows=rows, cols=cols, nnz=int(off[-1]), dtype=str(dt), bits=bits,
                                               pack=pack, cfg=str(cfg), worst=worst), flush=True)
                        return 1
                if pack:
                    m.drop_hot_columns()
        n_cases += 1
    print(f"fuzz ok: {n_cases} matrices, {n_runs} SpMVs", flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
