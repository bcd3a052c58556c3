"""Event timeline of the overlapped host SpMV (kernels._spmv_host_overlapped) on
C3 fp64: when x is up, when each row block's SpMV ends (compute stream) and when
its y download ends (copy stream), in ms from the call's start.

    python tools/host_overlap_timeline.py [blocks ...]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402
from paper_2301_04792_b200 import kernels  # noqa: E402
from paper_2301_04792_b200.device import cached_device_csr, host_to_device  # noqa: E402

d = lw.generate_rmat_csr(24, 16, seed=3, dtype="float64")
m = lw.CsrMatrix(d.rows, d.cols, d.row_offsets.cpu().numpy().astype(np.int64),
                 d.col_indices.cpu().numpy().astype(np.int64), d.values.cpu().numpy())
del d
x = np.random.default_rng(1).random(m.cols)
cfg = lw.ExecutorConfig()
dm = cached_device_csr(m, dtype="float64")
copy = torch.cuda.Stream()

for parts in [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]:
    blocks = kernels._row_blocks(dm, m.row_offsets, parts)
    stream = torch.cuda.current_stream()
    y = torch.empty(dm.rows, dtype=torch.float64, device="cuda")
    yh = torch.empty(dm.rows, dtype=torch.float64, pin_memory=True)
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        xd = host_to_device(x, dm.device, dm.dtype)
        ex = torch.cuda.Event(enable_timing=True)
        ex.record(stream)
        t_x = time.perf_counter()
        ev_s, ev_c = [], []
        for r0, r1, blk in blocks:
            kernels._launch(blk, xd, y[r0:r1], cfg, None, stream.cuda_stream)
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            ev_s.append(e)
            copy.wait_event(e)
            with torch.cuda.stream(copy):
                yh[r0:r1].copy_(y[r0:r1], non_blocking=True)
                c = torch.cuda.Event(enable_timing=True)
                c.record(copy)
                ev_c.append(c)
        t_l = time.perf_counter()
        copy.synchronize()
        t1 = time.perf_counter()
    print(f"blocks={len(blocks)} wall {1e3 * (t1 - t0):.3f} ms (host upload returns {1e3 * (t_x - t0):.3f},"
          f" launches done {1e3 * (t_l - t0):.3f}); device: x up {e0.elapsed_time(ex):.3f}; spmv ends "
          + " ".join(f"{e0.elapsed_time(e):.3f}" for e in ev_s) + "; copy ends "
          + " ".join(f"{e0.elapsed_time(c):.3f}" for c in ev_c))
