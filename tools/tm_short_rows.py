import os, sys, torch
sys.path.insert(0, '.')
import paper_2301_04792_b200 as lw
for name, m in [("C2u", lw.generate_random_csr(1_000_000, 1_000_000, 32_000_000, seed=2)),
                ("uni2^20", lw.generate_random_csr(1 << 20, 1 << 20, 16 << 20, seed=4))]:
    A = m.to_device("float32")
    x = torch.ones(A.cols, dtype=A.dtype, device="cuda")
    cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.THREAD_MAPPED)
    y = lw.spmv(A, x, cfg); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): lw.spmv(A, x, cfg, out=y)
    e1.record(); torch.cuda.synchronize()
    print(os.environ.get("LWB200_LIB", "")[-10:], name, round(e0.elapsed_time(e1) / 10, 4))
