"""Dev-container only: time the real reference (lanework numba, /root/reference) and
the oracle port (oracle/lw_oracle.c) on the same matrix and thread count, to show
the CPU baseline the bench reports is a faithful stand-in for the reference."""
import os, sys, time
sys.path.insert(0, '.')
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
import lanework as ref
from oracle import oracle
import paper_2301_04792_b200 as lwb

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
threads = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
off, col, val = oracle.rmat_csr(scale, 16, 3, lwb.rmat_thresholds(), threads=threads)
m = ref.CsrMatrix(len(off) - 1, len(off) - 1, off, col, val)
x = np.ones(m.cols)
for kind, ok in (("merge-path", ref.ScheduleKind.MERGE_PATH), ("thread-mapped", ref.ScheduleKind.THREAD_MAPPED)):
    cfg = ref.ExecutorConfig(schedule=ok, worker_threads=threads)
    ref.spmv(m, x, cfg)
    t = []
    for _ in range(5):
        t0 = time.perf_counter(); yr = ref.spmv(m, x, cfg); t.append(time.perf_counter() - t0)
    oracle.spmv(off, col, val, x, kind, lanes=32 * threads, threads=threads)
    u = []
    for _ in range(5):
        t0 = time.perf_counter(); yo = oracle.spmv(off, col, val, x, kind, lanes=32 * threads, threads=threads); u.append(time.perf_counter() - t0)
    print(f"scale {scale} nnz {m.nnz} {kind:14s} threads {threads}: reference numba {np.median(t)*1e3:8.1f} ms "
          f"({2*m.nnz/np.median(t)/1e9:.3f} GFLOP/s)  oracle port {np.median(u)*1e3:8.1f} ms ({2*m.nnz/np.median(u)/1e9:.3f} GFLOP/s)  "
          f"max|dy| {np.abs(yr-yo).max():.2e}")
