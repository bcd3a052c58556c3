"""Per-call host overhead of the device-operand API on a tiny matrix (the kernel
work is negligible, so this is Python + ctypes + launch cost)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402

m = lw.generate_random_csr(64, 64, 256, seed=1)
A = m.to_device("float32")
x = torch.ones(64, device="cuda")
y = torch.empty(64, device="cuda")
B = torch.ones(64, 8, device="cuda")
C = torch.empty(64, 8, device="cuda")
for kind in lw.ScheduleKind:
    cfg = lw.ExecutorConfig(schedule=kind)
    for name, fn in (("spmv", lambda: lw.spmv(A, x, cfg, out=y)), ("spmm", lambda: lw.spmm(A, B, cfg, out=C))):
        for _ in range(50):
            fn()
        torch.cuda.synchronize()
        n = 2000
        t = time.perf_counter()
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        print(f"{name} {kind.value:14s} {1e6 * (time.perf_counter() - t) / n:7.1f} us/call")
