import sys, torch, os
sys.path.insert(0, '.')
import numpy as np
import paper_2301_04792_b200 as lw
for name, m in [("pl1M", lw.generate_power_law_csr(1_000_000, 16.0, 1.1, seed=1)),
                ("pl2^20 s1.05", lw.generate_power_law_csr(1 << 20, 16.0, 1.05, seed=4))]:
    for dt in ("float32", "float64"):
        A = m.to_device(dt)
        x = torch.ones(A.cols, dtype=A.dtype, device="cuda")
        cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind.THREAD_MAPPED)
        y = lw.spmv(A, x, cfg); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): lw.spmv(A, x, cfg, out=y)
        e1.record(); torch.cuda.synchronize()
        print(os.environ.get("LWB200_LIB", "")[-10:], name, dt, round(e0.elapsed_time(e1) / 5, 3), "max row", int(np.diff(m.row_offsets).max()))
