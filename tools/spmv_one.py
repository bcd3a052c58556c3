"""A few back-to-back SpMVs of one BASELINE workload under one schedule, for an ncu
capture of that schedule's kernel (the bench_sweep matrices, same generators).

    python tools/spmv_one.py C2b group_block [fp32|fp64] [reps]     (C4 skew s: C4s<s>)
    schedules: thread_mapped, work_oriented, work_oriented_hot, group_warp, group_block
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2301_04792_b200 as lw  # noqa: E402

K = lw.ScheduleKind
SCHED = {"thread_mapped": (K.THREAD_MAPPED, 32), "work_oriented": (K.MERGE_PATH, 32),
         "work_oriented_hot": (K.MERGE_PATH, 32), "group_warp": (K.GROUP_MAPPED, 32),
         "group_block": (K.GROUP_MAPPED, 256)}


def matrix(name, dt):
    if name == "C1":
        return lw.generate_random_csr(10_000, 10_000, 1_000_000, seed=1).to_device(dt)
    if name == "C2b":
        return lw.generate_banded_device(1_000_000, 16, seed=2, dtype=dt)
    if name == "C2u":
        return lw.generate_uniform_device(1_000_000, 1_000_000, 32_000_000, seed=2, dtype=dt)
    if name.startswith("C4s"):   # C4 power-law matrix of the given skew, e.g. C4s1.05
        return lw.generate_power_law_csr(1 << 20, 16.0, float(name[3:]), seed=4).to_device(dt)
    if name == "C3":
        return lw.generate_rmat_csr(24, 16, seed=3, dtype=dt)
    raise SystemExit(f"unknown workload {name}")


def main():
    name, sched = sys.argv[1], sys.argv[2]
    dt = {"fp32": "float32", "fp64": "float64"}[sys.argv[3] if len(sys.argv) > 3 else "fp32"]
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    A = matrix(name, dt)
    if sched == "work_oriented_hot":
        A.pack_hot_columns()
    kind, gs = SCHED[sched]
    cfg = lw.ExecutorConfig(schedule=kind, group_size=gs)
    x = torch.rand(A.cols, device="cuda", dtype=A.values.dtype)
    for _ in range(reps):
        y = lw.spmv(A, x, cfg)
    torch.cuda.synchronize()
    print(name, sched, dt, A.rows, A.nnz, float(y.double().sum()))


if __name__ == "__main__":
    main()
