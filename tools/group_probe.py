import os, sys, torch
sys.path.insert(0, '.')
import paper_2301_04792_b200 as lw
mats = [("C2b", lw.generate_banded_device(1_000_000, 16, seed=1)),
        ("pl1M", lw.generate_power_law_csr(1_000_000, 16.0, 1.1, seed=1).to_device("float32")),
        ("C2u", lw.generate_random_csr(1_000_000, 1_000_000, 32_000_000, seed=2).to_device("float32")),
        ("C3", lw.generate_rmat_csr(24, 16, seed=3))]
for name, A in mats:
    x = torch.ones(A.cols, dtype=A.dtype, device="cuda")
    for gs in (32, 256):
        cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.GROUP_MAPPED, group_size=gs)
        y = lw.spmv(A, x, cfg); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): lw.spmv(A, x, cfg, out=y)
        e1.record(); torch.cuda.synchronize()
        print(os.environ.get("LWB200_LIB", "cur")[-10:], name, "gs", gs, round(e0.elapsed_time(e1) / 5, 3))
