"""One SSSP / BFS run for ncu launch lists: python tools/traversal_one.py sssp work_oriented [scale]"""
import sys

import torch

sys.path.insert(0, '.')
import paper_2301_04792_b200 as lwb  # noqa: E402

op, sched = sys.argv[1], sys.argv[2]
scale = int(sys.argv[3]) if len(sys.argv) > 3 else 22
A = lwb.generate_rmat_csr(scale, 16, seed=3, dtype="float64")
G = lwb.DeviceCsr(A.rows, A.cols, A.row_offsets, A.col_indices, A.values.abs())
src = int(torch.argmax(G.row_offsets[1:] - G.row_offsets[:-1]).item())
kind = {"work_oriented": lwb.ScheduleKind.MERGE_PATH, "thread_mapped": lwb.ScheduleKind.THREAD_MAPPED,
        "group_mapped": lwb.ScheduleKind.GROUP_MAPPED}[sched]
fn = lwb.sssp if op == "sssp" else lwb.bfs
cfg = lwb.ExecutorConfig(schedule=kind)
fn(G, src, cfg)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, passes = fn(G, src, cfg, return_passes=True)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(op, sched, scale, "passes", passes, "ms", round(sorted(ts)[1], 3))
