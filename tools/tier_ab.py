"""A/B of the work_oriented kernels on C3 (R-MAT 2^24 fp32): one-shot chunk
kernel (unpacked, hot-x packed) vs the persistent shared-memory tier kernel
(k_wo_tier) over tier sizes and group shapes. Every variant's y must be
bit-identical to the unpacked kernel's. One JSON line per variant."""
import json
import os
import sys

sys.path.insert(0, ".")
import torch

import paper_2301_04792_b200 as lwb

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
A = lwb.generate_rmat_csr(scale, 16, seed=3)
x = torch.rand(A.cols, device="cuda")
cfg = lwb.ExecutorConfig(schedule=lwb.ScheduleKind.WORK_ORIENTED)
alg = A.algorithmic_bytes()
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6554.0


def timeit(reps=30):
    y = lwb.spmv(A, x, cfg)
    for _ in range(5):
        lwb.spmv(A, x, cfg, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        lwb.spmv(A, x, cfg, out=y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, y


def emit(name, ms, y, ref, **kw):
    print(json.dumps({"variant": name, "ms": round(ms, 4), "gbs": round(alg / ms / 1e6, 1),
                      "frac_step": round(alg / ms / 1e6 / peak, 4),
                      "bit_identical": bool(torch.equal(y, ref)), **kw}), flush=True)


A.drop_hot_columns()
ms, ref = timeit()
emit("unpacked", ms, ref, ref)
for max_hot in [int(v) for v in os.environ.get("HOTS", "12288,24576,32768").split(",")]:
    A.drop_hot_columns()
    hx = A.pack_hot_columns(max_hot)
    os.environ["LW_WO_TIER"] = "0"
    ms, y = timeit()
    emit("packed-chunk", ms, y, ref, n_hot=hx.n_hot)
    os.environ["LW_WO_TIER"] = "1"
    for shape in [int(v) for v in os.environ.get("SHAPES", "0,1,2,3").split(",")]:
        os.environ["LW_WO_TIER_SHAPE"] = str(shape)
        for cap in [int(v) for v in os.environ.get("CAPS", "0,100000").split(",")]:
            os.environ["LW_WO_TIER_MAX"] = str(cap)
            ms, y = timeit()
            emit("tier", ms, y, ref, n_hot=hx.n_hot, shape=shape, tier_cap=cap)
