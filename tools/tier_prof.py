"""One C3 SpMV through the shared-memory tier kernel (k_wo_tier, 32 K hot
slots, 2 groups of 512) for an ncu capture."""
import os
import sys

sys.path.insert(0, ".")
import torch

import paper_2301_04792_b200 as lwb

A = lwb.generate_rmat_csr(24, 16, seed=3)
x = torch.rand(A.cols, device="cuda")
A.pack_hot_columns(int(os.environ.get("MAX_HOT", "32768")))
cfg = lwb.ExecutorConfig(schedule=lwb.ScheduleKind.WORK_ORIENTED)
for _ in range(4):
    lwb.spmv(A, x, cfg)
torch.cuda.synchronize()
