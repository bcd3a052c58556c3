"""One group_mapped (warp tiles) SpMV on C2b (banded 1M rows) and C2u (uniform 1M x 1M, 32M nnz),
fp32, for an ncu capture of the staged / cooperative warp kernels."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402

cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.GROUP_MAPPED, group_size=32)
for name in sys.argv[1:] or ["C2b", "C2u"]:
    if name == "C2b":
        A = lw.generate_banded_device(1_000_000, 16, seed=2, dtype="float32")
    else:
        A = lw.generate_random_csr(1_000_000, 1_000_000, 32_000_000, seed=2).to_device("float32")
    x = torch.ones(A.cols, device="cuda")
    for _ in range(3):
        y = lw.spmv(A, x, cfg)
    torch.cuda.synchronize()
    print(name, A.rows, A.nnz, float(y.sum()))
