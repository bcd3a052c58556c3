"""Where the drop-in host call spmv(CsrMatrix, ndarray) spends its time (C3 fp64):
pageable -> pinned copy of x, H2D, SpMV, D2H, each timed alone."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402
from paper_2301_04792_b200.device import cached_device_csr, device_to_host, host_to_device  # noqa: E402


def wall(f, n=10):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    return round(float(np.median(ts)) * 1e3, 3)


d = lw.generate_rmat_csr(24, 16, seed=3, dtype="float64")
m = lw.CsrMatrix(d.rows, d.cols, d.row_offsets.cpu().numpy().astype(np.int64),
                 d.col_indices.cpu().numpy().astype(np.int64), d.values.cpu().numpy())
x = np.random.default_rng(1).random(m.cols)
dm = cached_device_csr(m, dtype="float64")
xd = host_to_device(x, dm.device)
y = torch.empty(dm.rows, dtype=torch.float64, device="cuda")
stage = torch.empty(m.cols, dtype=torch.float64, pin_memory=True)
tx = torch.from_numpy(x)
print("threads", torch.get_num_threads())
print("pageable->pinned copy_ ms", wall(lambda: stage.copy_(tx)))
print("np.copyto into pinned ms", wall(lambda: np.copyto(stage.numpy(), x)))
print("H2D from pinned ms", wall(lambda: xd.copy_(stage, non_blocking=True)))
print("H2D pageable ms", wall(lambda: xd.copy_(tx)))
print("host_to_device ms", wall(lambda: host_to_device(x, dm.device)))
cfg = lw.ExecutorConfig()
print("spmv device ms", wall(lambda: lw.spmv(dm, xd, cfg, out=y)))
print("device_to_host ms", wall(lambda: device_to_host(y)))
print("spmv(CsrMatrix, ndarray) ms", wall(lambda: lw.spmv(m, x, cfg)))
