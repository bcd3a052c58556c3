"""Time one schedule on C2b / C2u / C3 / C4 skew 1.05 with int64 row offsets (the
layout of matrices with nnz >= 2^31), for A/B runs of library variants:
    LWB200_LIB=variants/x.so python tools/ab_off64.py [group_block]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402
from tools.spmv_one import SCHED, matrix  # noqa: E402


def main():
    sched = sys.argv[1] if len(sys.argv) > 1 else "group_block"
    kind, gs = SCHED[sched]
    cfg = lw.ExecutorConfig(schedule=kind, group_size=gs)
    out = []
    for name in ("C2b", "C2u", "C3", "C4s1.05"):
        for dt in ("float32", "float64"):
            A = matrix(name, dt)
            A = lw.DeviceCsr(A.rows, A.cols, A.row_offsets.to(torch.int64), A.col_indices, A.values)
            x = torch.rand(A.cols, device="cuda", dtype=A.values.dtype)
            y = lw.spmv(A, x, cfg)
            for _ in range(3):
                lw.spmv(A, x, cfg, out=y)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                lw.spmv(A, x, cfg, out=y)
            e1.record()
            torch.cuda.synchronize()
            out.append(f"{name}/{dt[5:]}:{e0.elapsed_time(e1) / 10:.4f}")
            del A
    print(" ".join(out), flush=True)


if __name__ == "__main__":
    main()
