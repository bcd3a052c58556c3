"""One SpMM configuration, for ncu: python tools/spmm_one.py C3 16 work_oriented [float32|float64]"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2301_04792_b200 as lwb  # noqa: E402

name, n, sched = sys.argv[1], int(sys.argv[2]), sys.argv[3]
dt = sys.argv[4] if len(sys.argv) > 4 else "float32"
A = (lwb.generate_random_csr(1_000_000, 1_000_000, 32_000_000, seed=2).to_device(dt)
     if name == "C2u" else lwb.generate_rmat_csr(24 if name == "C3" else 22, 16, seed=3, dtype=dt))
kind = {"work_oriented": lwb.ScheduleKind.MERGE_PATH, "thread_mapped": lwb.ScheduleKind.THREAD_MAPPED,
        "group_mapped": lwb.ScheduleKind.GROUP_MAPPED}[sched]
B = torch.ones((A.cols, n), dtype=A.dtype, device=A.device)
C = torch.empty((A.rows, n), dtype=A.dtype, device=A.device)
cfg = lwb.ExecutorConfig(schedule=kind)
for _ in range(3):
    lwb.spmm(A, B, cfg, out=C)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lwb.spmm(A, B, cfg, out=C)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(name, n, sched, dt, "ms", round(sorted(ts)[2], 3))
