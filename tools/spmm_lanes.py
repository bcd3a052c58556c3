import sys, torch
sys.path.insert(0, '.')
import paper_2301_04792_b200 as lwb
for name in ["C2u", "C3"]:
    if name == "C2u":
        A = lwb.generate_random_csr(1_000_000, 1_000_000, 32_000_000, seed=2).to_device("float32")
    else:
        A = lwb.generate_rmat_csr(24, 16, seed=3)
    n = 16
    B = torch.ones((A.cols, n), dtype=A.dtype, device=A.device)
    C = torch.empty((A.rows, n), dtype=A.dtype, device=A.device)
    total = A.rows + A.nnz
    for items in [1024, 512, 256, 128, 64]:
        lanes = (total + items - 1) // items
        cfg = lwb.ExecutorConfig(schedule=lwb.ScheduleKind.MERGE_PATH, lanes=lanes)
        lwb.spmm(A, B, cfg, out=C); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): lwb.spmm(A, B, cfg, out=C)
        e1.record(); torch.cuda.synchronize()
        print(name, "items", items, "ms", round(e0.elapsed_time(e1) / 5, 3), flush=True)
    del A, B, C; torch.cuda.empty_cache()
