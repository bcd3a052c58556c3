"""Headline benchmark: work_oriented (merge-path) SpMV on a 2^24-row R-MAT CSR, fp32.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--schedule work_oriented|thread_mapped|group_warp|group_block]
                    [--scale 24] [--dtype fp32|fp64]

One step = one y = A x over the whole matrix with inputs resident in HBM (the
matrix is 2.2 GB fp32, far larger than the 126 MB L2, so no flush is needed
between steps; x (64 MB) may stay L2-resident across steps, as it would in an
iterated SpMV). Timed with CUDA events on the launching stream, bracketed by a
barrier + synchronize, max over ranks. Metric = GFLOP/s = 2*nnz / t.

N > 1 (torchrun, one rank per GPU): the same matrix is built on every rank,
split into nnz-balanced row shards (x replicated) and each rank times its own
shard; value = 2*nnz_total / max_rank(t) — total work fixed, "scaling": "strong".

e2e (the headline against the reference arm): the same SpMV through the C ABI
with HOST x and y — per step x is copied in from pinned memory, lw_spmv runs on
the resident matrix (the operator is uploaded once, like a model's weights) and
y is copied back, all inside the CUDA-event-timed region; e2e_cold also uploads
the whole CSR every call (lw_spmv_host), which is PCIe-bound.

--impl reference times the reference's CPU algorithm (the C oracle port of
lanework's numba merge-path loop, fp64/int64 like the reference, all host
threads, lanes = 32 x threads — the reference CLI's configuration) on the same
matrix generated on the host; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SpMV GFLOP/s (work_oriented merge-path, fp32, 2^24-row R-MAT CSR)"
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--schedule", default="work_oriented",
                    choices=["work_oriented", "thread_mapped", "group_warp", "group_block"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--seed", type=int, default=3)
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--hot-x", default="auto", choices=["auto", "on", "off"],
                    help="work_oriented: hot-x column packing (DESIGN.md 4e); auto = on (fp32 and fp64)")
    ap.add_argument("--max-hot", type=int, default=0, help="hot-x slots (0 = library default)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="spmv", choices=["spmv", "power"],
                    help="spmv: one y=Ax per step (C3 headline); power: C5 power iteration")
    ap.add_argument("--iters", type=int, default=20, help="power iterations per step (C5)")
    ap.add_argument("--graph", action="store_true",
                    help="power mode: capture the iterations once into a CUDA graph and replay it")
    ap.add_argument("--fused", action="store_true",
                    help="power mode: all-gather fused into the SpMV (peer/multicast row writes "
                         "into symmetric-memory buffers) instead of NCCL")
    ap.add_argument("--chunks", type=int, default=0,
                    help="power mode: row chunks per shard whose all-gathers overlap the next "
                         "chunk's SpMV (0 = 4 when N > 1, else 1)")
    ap.add_argument("--items", type=int, default=0,
                    help="work_oriented items per lane (0 = library default)")
    ap.add_argument("--balance", default="cost", choices=["cost", "work", "nnz"],
                    help="N > 1 row split: nnz + 1.75 rows (measured shard cost, default), rows + nnz "
                         "(merge-path tiles) or nnz balanced (distributed.row_bounds)")
    ap.add_argument("--relabel", default="on", choices=["on", "off"],
                    help="power mode: symmetric degree relabeling of the C5 operator (one-time)")
    ap.add_argument("--no-fp64", action="store_true", help="skip the fp64 C3 leg")
    ap.add_argument("--no-power", action="store_true", help="skip the C5 power-iteration leg")
    ap.add_argument("--power-scale", type=int, default=26, help="R-MAT scale of the C5 leg")
    ap.add_argument("--power-seed", type=int, default=5, help="R-MAT seed of the C5 leg")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch path only: rendezvous + one gloo all-reduce, no device work")
    return ap.parse_args()


def ncu_traffic(workload: str, dtype: str, schedule: str):
    """DRAM bytes per launch of the dominant kernel from the newest committed
    ncu --set full capture (profiles/*/ncu_traffic.json) for this workload."""
    best = None
    for f in sorted((ROOT / "profiles").glob("*/ncu_traffic*.json")):
        try:
            d = json.loads(f.read_text())
        except Exception:
            continue
        if d.get("workload") == workload and d.get("dtype") == dtype and d.get("schedule") == schedule:
            best = (int(d["traffic_bytes_per_launch"]), str(f.relative_to(ROOT)))
    return best


def peaks():
    try:
        d = json.loads(PEAKS_FILE.read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML every ~20 ms
    while the timed region runs (the same counters nvidia-smi's
    clocks.sm / clocks_event_reasons.* report)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period_s: float = 0.005):
        self.index = index
        self.period = period_s
        self.samples = []
        self.reason_bits = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.error = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        except Exception as exc:  # pragma: no cover - depends on the box
            self.error = repr(exc)
        return self

    def _sample(self):
        nv = self._nv
        self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
        self.reason_bits |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)

    def _loop(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception as exc:  # pragma: no cover
                self.error = repr(exc)
                return
            self._stop.wait(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0,
                    "error": self.error}
        reasons = sorted(k for k, bit in self.REASONS.items() if self.reason_bits & bit)
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------------------------------
def reference_arm(args):
    """Reference CPU algorithm (oracle port), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle
    from paper_2301_04792_b200.sparse import rmat_thresholds

    threads = oracle.default_threads()
    t0 = time.time()
    off, col, val = oracle.rmat_csr(args.scale, args.edge_factor, args.seed, rmat_thresholds(),
                                    threads=threads)
    if args.dtype == "fp32":
        val = val.astype(np.float32).astype(np.float64)
    gen_s = time.time() - t0
    rows = off.size - 1
    nnz = int(off[-1])
    x = np.ones(rows, dtype=np.float64)
    lanes = 32 * threads
    iters = args.iters if args.mode == "power" else 1

    def step():
        if args.mode != "power":
            oracle.spmv(off, col, val, x, "merge-path", lanes=lanes, threads=threads)
            return
        v = np.full(rows, 1.0 / np.sqrt(rows))
        for _ in range(iters):
            yv = oracle.spmv(off, col, val, v, "merge-path", lanes=lanes, threads=threads)
            v = yv / np.linalg.norm(yv)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        step()
        times.append(time.perf_counter() - t)
    sec = float(np.mean(times))     # whole job: K steps / their total time
    gflops = 2.0 * nnz * iters / sec / 1e9
    sample = (f"full R-MAT scale {args.scale} matrix ({rows} rows, {nnz} nnz), merge-path, "
              f"fp64/int64, {threads} threads, {lanes} lanes, mean of {args.steps} runs")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gflops, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": run_config(args, rows, nnz, 1),
        "cpu_baseline": {"value": round(gflops, 4), "unit": "GFLOP/s", "cores": threads,
                         "kind": "port", "sample": sample, "host": host_cpu(),
                         "median_ms": round(float(np.median(times)) * 1e3, 3)},
        "e2e": {"value": round(gflops, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "generation_s": round(gen_s, 2),
    }
    if args.mode != "power":
        line["reference_package"] = time_lanework(off, col, val, x, threads)
    print(json.dumps(line), flush=True)


def time_lanework(off, col, val, x, threads) -> dict:
    """lanework itself (baseline/_ref, installed offline from the reference's
    source; numba backend) on the same arrays: lanework.spmv(m, x,
    ExecutorConfig(merge-path, worker_threads=all)) — the reference CLI's call —
    warm-up (JIT) then the median of 5 (cli.py:137-145). Reported beside the
    port, which is faster than lanework here, so the ratios the
    driver computes against the port understate the speed-up over the reference."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "lanework").is_dir():
        return {"unavailable": "baseline/_ref/lanework not installed"}
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/lw_numba_cache")
    sys.path.insert(0, str(ref))
    try:
        import lanework
    except Exception as exc:  # pragma: no cover - depends on the box
        return {"unavailable": f"import failed: {exc!r}"}
    finally:
        sys.path.remove(str(ref))
    try:
        rows = off.size - 1
        m = lanework.CsrMatrix(rows, rows, off, col, val)
        cfg = lanework.ExecutorConfig(schedule=lanework.ScheduleKind.MERGE_PATH,
                                      worker_threads=threads)
        t = time.perf_counter()
        lanework.spmv(m, x, cfg)
        first = time.perf_counter() - t
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            lanework.spmv(m, x, cfg)
            ts.append(time.perf_counter() - t)
        sec = float(np.median(ts))
        return {"value": round(2.0 * int(off[-1]) / sec / 1e9, 4), "unit": "GFLOP/s",
                "ms_per_step": round(sec * 1e3, 2), "first_call_ms": round(first * 1e3, 1),
                "backend": lanework.backend_name(), "worker_threads": threads, "lanes": cfg.lanes,
                "sample": "lanework.spmv on the full matrix, median of 5 after one warm-up call"}
    except Exception as exc:  # pragma: no cover
        return {"unavailable": f"lanework.spmv failed: {exc!r}"}


def run_config(args, rows, nnz, world) -> dict:
    """The workload description both arms share (same keys, same values)."""
    return {"workload": f"rmat{args.scale}-ef{args.edge_factor}-seed{args.seed}",
            "schedule": args.schedule, "rows": rows, "nnz": nnz,
            "parallelism": f"rows{world}" if world > 1 else "single"}


# ---------------------------------------------------------------------------------------
def setup_ranks():
    """(world, rank, local, dev) with the process group initialised for N > 1:
    NCCL over NVLink, one rank per GPU. LW_BENCH_SHARE_GPU=1 (code-path check
    only, never a measurement) puts every rank on cuda:0 over gloo, so the N > 1
    path runs on a one-GPU box."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    share = os.environ.get("LW_BENCH_SHARE_GPU") == "1"
    local = 0 if share else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    return world, rank, local, dev


def power_arm(args):
    """--mode power: the C5 line alone (see power_measure)."""
    import torch.distributed as dist

    world, rank, local, dev = setup_ranks()
    line = power_measure(args, world, rank, local, dev, args.power_scale, args.power_seed)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def power_measure(args, world, rank, local, dev, scale, seed):
    """C5: x <- A x / ||A x|| for --iters iterations on nnz-balanced row shards.
    One step = the whole iteration sequence; each iteration is the shard's
    work_oriented SpMV plus one NCCL all-gather of the uneven y shards (row
    chunks whose all-gathers overlap the next chunk's SpMV when N > 1), or with
    --fused the all-gather folded into the SpMV's row stores. Returns the line."""
    import torch
    import torch.distributed as dist

    import paper_2301_04792_b200 as lwb
    from paper_2301_04792_b200.distributed import RowShard, power_iteration, row_bounds

    dtype = "float32" if args.dtype == "fp32" else "float64"
    full = lwb.generate_rmat_csr(scale, args.edge_factor, seed, dtype=dtype, device=dev)
    n, nnz_total = full.rows, full.nnz
    # one-time operator preparation (like the matrix upload, outside the timed
    # region): symmetric degree relabeling P A P^T (hot x entries become a dense,
    # cache-resident prefix), then the nnz-balanced row shard
    relabel = args.relabel == "on" and not (args.fused or args.graph)
    prep_ms = {}
    R = None
    if relabel:
        torch.cuda.synchronize()
        t_r = time.perf_counter()
        R = full.degree_relabel()
        torch.cuda.synchronize()
        prep_ms["relabel"] = round((time.perf_counter() - t_r) * 1e3, 1)
        full = R.matrix
    bounds = row_bounds(full.row_offsets.cpu().numpy(), world, args.balance)
    shard = RowShard(bounds, rank)
    A = full.row_slice(shard.r0, shard.r1)
    A = lwb.DeviceCsr(A.rows, A.cols, A.row_offsets.clone(), A.col_indices.clone(), A.values.clone())
    del full
    torch.cuda.empty_cache()
    cfg = lwb.ExecutorConfig(schedule=lwb.ScheduleKind.MERGE_PATH)
    y_local = torch.empty(A.rows, dtype=A.dtype, device=dev)
    chunks = args.chunks or (4 if world > 1 else 1)
    # hot-x packing of every SpMV operand (one-time, before warm-up)
    hot = args.hot_x in ("on", "auto")
    spmv_ev = []
    layout = None
    if not (args.fused or args.graph):
        # in-place gather layout: operator columns renamed into the all-gather
        # buffer, so each iteration is SpMV -> in-place all-gather -> norm -> scale
        from paper_2301_04792_b200.distributed import GatherLayout, power_iteration_inplace

        torch.cuda.synchronize()
        t_l = time.perf_counter()
        # exact (unpadded) layout over NCCL: uneven per-rank pieces, no padding
        exact = world > 1 and dist.get_backend() == "nccl"
        layout = GatherLayout(bounds, chunks, exact=exact)
        A = layout.remap_columns(A)
        pos_t = layout.pos_on(dev)
        # buffer form -> original numbering in one gather (relabel composed in)
        final_idx = pos_t if R is None else pos_t.index_select(0, R.rank.to(torch.int64))
        slices = {}
        for k in range(layout.chunks):
            _, _, r0, r1 = layout.slot(rank, k)
            Ak = A if (r0, r1) == (0, A.rows) else A.row_slice(r0, r1)
            if Ak.nnz and (Ak.col_indices.data_ptr() % 32 or Ak.values.data_ptr() % 32):
                # a view starting mid-sector would run the chunk kernel without its
                # 32-byte vector loads: give the chunk its own aligned copy
                Ak = lwb.DeviceCsr(Ak.rows, Ak.cols, Ak.row_offsets, Ak.col_indices.clone(),
                                   Ak.values.clone())
            if hot:
                Ak.pack_hot_columns(args.max_hot or None)
            slices[(r0, r1)] = Ak
        torch.cuda.synchronize()
        prep_ms["layout_and_hotx"] = round((time.perf_counter() - t_l) * 1e3, 1)

        def slot_spmv(x, r0, r1, out):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            lwb.spmv(slices[(r0, r1)], x, cfg, out=out)
            e1.record()
            spmv_ev.append((e0, e1))
    elif hot:
        A.pack_hot_columns(args.max_hot or None)

    if args.graph:
        from paper_2301_04792_b200.distributed import power_iteration_graph

        def plain_spmv(x):
            lwb.spmv(A, x, cfg, out=y_local)
            return y_local

        graphs = {}

        def run_iters(k):
            if k not in graphs:
                graphs[k] = power_iteration_graph(plain_spmv, n, shard, k, dtype=A.dtype, device=dev)
            return graphs[k]()
    elif args.fused:
        from paper_2301_04792_b200.distributed import power_iteration_fused

        def run_iters(k):
            return power_iteration_fused(A, n, shard, k)
    else:
        def run_iters(k):
            xb, norms = power_iteration_inplace(slot_spmv, layout, k, rank=rank, dtype=A.dtype, device=dev)
            return xb.index_select(0, final_idx), norms

    for _ in range(max(args.warmup, 3)):
        run_iters(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    spmv_ev.clear()
    with ClockSampler(local) as clocks:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            x, norms = run_iters(args.iters)
        t1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1) / args.steps
    spmv_ms = sum(a.elapsed_time(b) for a, b in spmv_ev) / args.steps
    if world > 1:
        t = torch.tensor([ms, spmv_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, spmv_ms = float(t[0]), float(t[1])
    gflops = 2.0 * nnz_total * args.iters / (ms * 1e-3) / 1e9
    line = {
        "metric": (f"power iteration GFLOP/s ({args.iters} iters, work_oriented SpMV "
                   + ("with the y all-gather fused into its row writes)" if args.fused
                      else "+ NCCL y all-gather)")),
        "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32" if args.dtype == "fp32" else "f64",
        "data": "synthetic",
        "config": {"workload": f"rmat{scale}-ef{args.edge_factor}-seed{seed}-power{args.iters}",
                   "rows": n, "nnz": nnz_total, "parallelism": f"rows{world}" if world > 1 else "single",
                   "row_split": args.balance if world > 1 else None,
                   "overlap_chunks": 0 if (args.fused or args.graph) else chunks,
                   "fused_allgather": bool(args.fused), "cuda_graph": bool(args.graph),
                   "x_layout": ("degree-relabeled P A P^T (DESIGN.md 4f)" if relabel else "as generated")
                               + (" + hot-x packed (DESIGN.md 4e)" if hot else ""),
                   "gather": (("exact in-place all-gather (uneven pieces)" if layout.exact else
                               "in-place all-gather layout") if layout is not None else
                              "fused into the SpMV row stores" if args.fused else "CUDA graph")},
        "allgather_mb_per_gpu_per_iter": (None if layout is None or world == 1 else round(
            ((layout.size - shard.rows) if layout.exact else (layout.size - sum(layout.widths)))
            * A.values.element_size() / 1e6, 1)),
        "one_time_prep_ms": prep_ms,
        "breakdown_ms": None if (args.fused or args.graph) else {"spmv_max_rank": round(spmv_ms, 3),
                                                 "allgather_normalise": round(ms - spmv_ms, 3)},
        "final_norm": norms[-1] if norms else None,
        "gpu_launches": ((3 + (hot and args.fused and world > 1)) * (1 if args.fused else chunks) + 3)
                        * args.iters * args.steps,
        "clocks": clocks.summary(),
    }
    del A
    torch.cuda.empty_cache()
    return line


# ---------------------------------------------------------------------------------------
def our_arm(args):
    import torch
    import torch.distributed as dist

    import paper_2301_04792_b200 as lwb
    from paper_2301_04792_b200 import _lib
    from paper_2301_04792_b200.device import current_stream
    from paper_2301_04792_b200.distributed import row_bounds

    world, rank, local, dev = setup_ranks()

    def barrier():
        if world > 1:
            dist.barrier()

    dtype = "float32" if args.dtype == "fp32" else "float64"
    full = lwb.generate_rmat_csr(args.scale, args.edge_factor, args.seed, dtype=dtype, device=dev)
    nnz_total = full.nnz
    rows_total = full.rows
    if world > 1:
        bounds = row_bounds(full.row_offsets.cpu().numpy(), world, args.balance)
        A = full.row_slice(int(bounds[rank]), int(bounds[rank + 1]))
        A = lwb.DeviceCsr(A.rows, A.cols, A.row_offsets.clone(), A.col_indices.clone(),
                          A.values.clone())
        del full
        torch.cuda.empty_cache()
    else:
        A = full
    x = torch.ones(A.cols, dtype=A.dtype, device=dev)
    y = torch.empty(A.rows, dtype=A.dtype, device=dev)

    sched = {"work_oriented": lwb.ScheduleKind.MERGE_PATH,
             "thread_mapped": lwb.ScheduleKind.THREAD_MAPPED,
             "group_warp": lwb.ScheduleKind.GROUP_MAPPED,
             "group_block": lwb.ScheduleKind.GROUP_MAPPED}[args.schedule]
    gs = 256 if args.schedule == "group_block" else 32
    cfg = lwb.ExecutorConfig(schedule=sched, group_size=gs)
    lib = _lib.load()
    Ac = A.c_struct()
    stream = torch.cuda.current_stream(dev)
    sp = current_stream(dev)
    ws_bytes = lib.lw_spmv_workspace(_lib.LW_MERGE_PATH, A.rows, A.nnz, 0, Ac.dtype)
    ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)
    launches_per_step = 3 if sched is lwb.ScheduleKind.MERGE_PATH else 1
    if args.schedule == "group_warp":   # staged + cooperative pair on >= 4 blocks per SM
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        launches_per_step = 2 if -(-A.rows // 32) >= 4 * sms else 1
    lanes = 0
    if args.items and sched is lwb.ScheduleKind.MERGE_PATH:
        lanes = -(-(A.rows + A.nnz) // args.items)
        ws_bytes = lib.lw_spmv_workspace(_lib.LW_MERGE_PATH, A.rows, A.nnz, lanes, Ac.dtype)
        ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device=dev)

    # hot-x column packing (one-time inspector, outside the timed region like the
    # matrix upload): work_oriented, both dtypes by default
    hx, hx_build_ms = None, None
    if sched is lwb.ScheduleKind.MERGE_PATH and args.hot_x in ("on", "auto"):
        torch.cuda.synchronize()
        t_b = time.perf_counter()
        hx = A.pack_hot_columns(args.max_hot or None)
        torch.cuda.synchronize()
        hx_build_ms = (time.perf_counter() - t_b) * 1e3
        hx_ws_bytes = lib.lw_spmv_work_oriented_hotx_workspace(A.rows, A.nnz, lanes, hx.n_hot, Ac.dtype)
        hx_ws = torch.empty(max(hx_ws_bytes, 256), dtype=torch.uint8, device=dev)
        Hc = hx.packed.c_struct()
        hot_ptr = hx.hot_cols.data_ptr() if hx.n_hot else None

    # one step, with the dominant kernel bracketed by events
    ev = []

    def phase(mask, packed):
        if packed:
            return lib.lw_spmv_work_oriented_hotx_phases(Hc, hot_ptr, hx.n_hot, x.data_ptr(), y.data_ptr(),
                                                         lanes, hx_ws.data_ptr(), hx_ws.numel(), mask, sp)
        return lib.lw_spmv_work_oriented_phases(Ac, x.data_ptr(), y.data_ptr(), lanes, ws.data_ptr(),
                                                ws.numel(), mask, sp)

    def step(record, packed=None):
        packed = hx is not None if packed is None else packed
        if sched is lwb.ScheduleKind.MERGE_PATH:
            _lib.check(phase(1, packed), "p1")
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            _lib.check(phase(2, packed), "p2")
            if record:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                ev.append((e0, e1))
            _lib.check(phase(4, packed), "p3")
        else:
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            lwb.spmv(A, x, cfg, out=y)
            if record:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                ev.append((e0, e1))

    for _ in range(max(args.warmup, 3)):
        step(False)
    torch.cuda.synchronize()
    # pass A: whole steps timed back to back (the headline value)
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            step(False)
        t1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = t0.elapsed_time(t1)
    # pass B: same steps with the dominant kernel bracketed (events add a little gap)
    ev.clear()
    for _ in range(args.steps):
        step(True)
    torch.cuda.synchronize()
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    if hx is not None:
        y_packed = y.clone()
        # pass C: the unpacked kernel on the same inputs (bit-identical y), for the record
        for _ in range(3):
            step(False, packed=False)
        torch.cuda.synchronize()
        u0 = torch.cuda.Event(enable_timing=True)
        u1 = torch.cuda.Event(enable_timing=True)
        u0.record(stream)
        for _ in range(args.steps):
            step(False, packed=False)
        u1.record(stream)
        torch.cuda.synchronize()
        ms_unpacked = u0.elapsed_time(u1) / args.steps
        ev.clear()
        for _ in range(args.steps):
            step(True, packed=False)
        torch.cuda.synchronize()
        kern_unpacked = float(np.mean([a.elapsed_time(b) for a, b in ev]))
        same = bool(torch.equal(y, y_packed))

    ms = ms_total / args.steps
    if world > 1:
        t = torch.tensor([ms, kern_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kern_ms = float(t[0]), float(t[1])
    gflops = 2.0 * nnz_total / (ms * 1e-3) / 1e9

    # algorithmic bytes of the dominant kernel for this rank's shard
    alg_bytes = A.algorithmic_bytes()
    sv = A.values.element_size()
    gather_bytes = alg_bytes - A.cols * sv + A.nnz * sv
    hbm, hbm_src = peaks()
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    workload = f"rmat{args.scale}-ef{args.edge_factor}-seed{args.seed}"
    tr_key = args.schedule + ("+hotx" if hx is not None else "")
    tr = ncu_traffic(workload, "f32" if args.dtype == "fp32" else "f64", tr_key) if world == 1 else None
    traffic = tr[0] if tr else None
    line = {
        "metric": METRIC, "value": round(gflops, 3), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if args.dtype == "fp32" else "f64", "data": "synthetic",
        "config": run_config(args, rows_total, nnz_total, world),
        "notes": {"l2": "inputs > L2 (2.2 GB matrix streamed per step); no flush",
                  **({"row_split": f"{args.balance}-balanced rows (distributed.row_bounds)"} if world > 1 else {})},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
                     "unit": "GB/s", "frac": round(achieved / hbm, 4), "traffic": traffic,
                     "kernel": "k_wo_chunk" if sched is lwb.ScheduleKind.MERGE_PATH else args.schedule,
                     "kernel_ms": round(kern_ms, 4), "alg_bytes": alg_bytes,
                     "peak_source": hbm_src, "frac_of_8TBps": round(achieved / 8000.0, 4),
                     "traffic_source": tr[1] if tr else None,
                     # SURVEY §8(d) upper model: every atom gathers its own x value
                     "achieved_gather_every_nnz": round(gather_bytes / (kern_ms * 1e-3) / 1e9, 1),
                     "frac_gather_every_nnz": round(gather_bytes / (kern_ms * 1e-3) / 1e9 / hbm, 4)},
        "hbm_gbs_step": round(alg_bytes / (ms * 1e-3) / 1e9, 1),
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks.summary(),
    }
    if hx is not None:
        line["notes"]["x_layout"] = (f"hot-x packed: {hx.n_hot} most gathered columns in a dense "
                                      f"per-call copy kept in L1 (DESIGN.md 4e); one-time inspector "
                                      f"{hx_build_ms:.1f} ms outside the timed region")
        line["roofline"]["kernel"] = "k_wo_chunk (hot-x packed; the pack rides on the partition launch)"
        line["unpacked"] = {"ms_per_step": round(ms_unpacked, 4), "kernel_ms": round(kern_unpacked, 4),
                            "value": round(2.0 * nnz_total / (ms_unpacked * 1e-3) / 1e9, 3),
                            "frac": round(alg_bytes / (kern_unpacked * 1e-3) / 1e9 / hbm, 4),
                            "y_bit_identical": same}

    # e2e through the C ABI with HOST x and y (pinned), copies inside the timed
    # region; the matrix is the resident operator (uploaded once, like weights).
    # e2e_cold additionally uploads the whole CSR every call (lw_spmv_host).
    # At N > 1 every rank runs the same loop on its shard (full x in, its rows of
    # y out); the job's time is the slowest rank's and the bytes are summed.
    if not args.no_e2e:
        barrier()
        e2e = e2e_resident(A, args, lib, dev, nnz_total)
        if world > 1:
            t = torch.tensor([e2e["ms_per_step"], e2e["h2d_bytes_per_step"],
                              e2e["d2h_bytes_per_step"]], dtype=torch.float64, device=dev)
            tmax, tsum = t.clone(), t.clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
            e2e_ms = float(tmax[0])
            e2e.update({"value": round(2.0 * nnz_total / (e2e_ms * 1e-3) / 1e9, 3),
                        "ms_per_step": round(e2e_ms, 3), "h2d_bytes_per_step": int(tsum[1]),
                        "d2h_bytes_per_step": int(tsum[2]),
                        "path": e2e["path"] + f"; {world} ranks, max over ranks"})
        line["e2e"] = e2e
        if world == 1:
            line["e2e_cold"] = e2e_host(A, args, lib, dev, nnz_total)
    if hx is not None:
        # one-time inspector vs per-call saving: SpMVs after which packing has paid
        saved = ms_unpacked - ms
        line["notes"]["hotx_break_even_spmvs"] = (round(hx_build_ms / saved, 1) if saved > 0
                                                   else None)
    if not args.no_fp64 and args.dtype == "fp32" and sched is lwb.ScheduleKind.MERGE_PATH:
        line["fp64"] = fp64_leg(A, args, lib, dev, world, nnz_total, hbm)
    if not args.no_e2e and world == 1 and sched is lwb.ScheduleKind.MERGE_PATH:
        line["e2e_api"] = e2e_api(A, args, nnz_total)
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline(A, args)
    if not args.no_power and args.mode == "spmv":
        del A, x, y, ws
        hx = None
        torch.cuda.empty_cache()
        barrier()
        line["power"] = power_measure(args, world, rank, local, dev, args.power_scale, args.power_seed)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line), flush=True)


def fp64_leg(A, args, lib, dev, world, nnz_total, hbm):
    """The same C3 matrix with fp64 values (the reference's only precision,
    sparse.py:55-58): work_oriented kernel, hot-x packed like the headline (and
    unpacked beside it, y compared bit for bit), timed like the headline."""
    import torch
    import torch.distributed as dist

    import paper_2301_04792_b200 as lwb

    A64 = A.astype("float64")
    x = torch.ones(A64.cols, dtype=torch.float64, device=dev)
    y = torch.empty(A64.rows, dtype=torch.float64, device=dev)
    cfg = lwb.ExecutorConfig(schedule=lwb.ScheduleKind.MERGE_PATH)

    def timed():
        for _ in range(max(args.warmup, 3)):
            lwb.spmv(A64, x, cfg, out=y)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            lwb.spmv(A64, x, cfg, out=y)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        if world > 1:
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t[0])
        return ms

    ms_plain = timed()
    y_plain = y.clone()
    packed = args.hot_x in ("on", "auto")
    ms = ms_plain
    if packed:
        A64.pack_hot_columns(args.max_hot or None)
        ms = timed()
    alg = A64.algorithmic_bytes()
    out = {"dtype": "f64", "ms_per_step": round(ms, 4),
           "value": round(2.0 * nnz_total / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
           "hbm_gbs_step": round(alg / (ms * 1e-3) / 1e9, 1),
           "frac_step": round(alg / (ms * 1e-3) / 1e9 / hbm, 4), "alg_bytes": alg,
           "path": ("lw_spmv_work_oriented_hotx" if packed else "lw_spmv_work_oriented")
                   + " (fp64 values and x, int32 columns), 3 launches per step"}
    if packed:
        out["unpacked"] = {"ms_per_step": round(ms_plain, 4),
                           "value": round(2.0 * nnz_total / (ms_plain * 1e-3) / 1e9, 3),
                           "y_bit_identical": bool(torch.equal(y, y_plain))}
    del A64, x, y, y_plain
    torch.cuda.empty_cache()
    return out


def e2e_api(A, args, nnz_total):
    """The call a lanework user makes, unchanged: lw.spmv(CsrMatrix, ndarray)
    with the reference's defaults (kernels.py:57-69: merge-path, fp64 arithmetic,
    NumPy float64 x in and a new NumPy float64 y out). The CsrMatrix's device copy
    is cached by the package after the first call (like numba's compiled kernel
    in the reference); every timed call uploads x, runs the SpMV and returns y on
    the host, timed by the wall clock around the synchronous call."""
    import paper_2301_04792_b200 as lwb
    from paper_2301_04792_b200.device import drop_device_cache

    m = lwb.CsrMatrix(A.rows, A.cols, A.row_offsets.cpu().numpy().astype(np.int64),
                      A.col_indices.cpu().numpy().astype(np.int64),
                      A.values.cpu().numpy().astype(np.float64))
    x = np.ones(A.cols)
    for _ in range(3):
        y = lwb.spmv(m, x)
    ts = []
    for _ in range(max(5, min(args.steps, 20))):
        t = time.perf_counter()
        y = lwb.spmv(m, x)
        ts.append(time.perf_counter() - t)
    sec = float(np.median(ts))
    drop_device_cache(m)
    return {"value": round(2.0 * nnz_total / sec / 1e9, 3), "unit": "GFLOP/s",
            "ms_per_step": round(sec * 1e3, 3), "dtype": "f64", "steps": len(ts),
            "h2d_bytes_per_step": int(x.nbytes), "d2h_bytes_per_step": int(y.nbytes),
            "path": "paper_2301_04792_b200.spmv(CsrMatrix, numpy x) -> numpy y, default "
                    "ExecutorConfig (merge-path), fp64; median wall time of the synchronous call"}


def e2e_resident(A, args, lib, dev, nnz_total):
    """Per step: x host->device (pinned), lw_spmv (C ABI, work_oriented) on the
    resident matrix, y device->host (pinned). Steps are pipelined the way a
    serving loop would run them: copy-in, compute and copy-out on three streams
    with double-buffered x/y, so step i+1's x upload and step i-1's y download
    (the PCIe link is full duplex) overlap step i's SpMV. CUDA events bracket
    the whole sequence, every step's copies included."""
    import torch

    from paper_2301_04792_b200 import _lib

    h_x = [torch.ones(A.cols, dtype=A.dtype).pin_memory() for _ in range(2)]
    h_y = [torch.empty(A.rows, dtype=A.dtype).pin_memory() for _ in range(2)]
    d_x = [torch.empty(A.cols, dtype=A.dtype, device=dev) for _ in range(2)]
    d_y = [torch.empty(A.rows, dtype=A.dtype, device=dev) for _ in range(2)]
    Ac = A.c_struct()
    s_in, s_comp, s_out = (torch.cuda.Stream(dev) for _ in range(3))
    hx = A.hot_columns()   # the packed operator when the bench built one (hot-x)
    if hx is not None:
        Hc = hx.packed.c_struct()
        hot_ptr = hx.hot_cols.data_ptr() if hx.n_hot else None
        ws_b = lib.lw_spmv_work_oriented_hotx_workspace(A.rows, A.nnz, 0, hx.n_hot, Ac.dtype)
    else:
        ws_b = lib.lw_spmv_workspace(_lib.LW_MERGE_PATH, A.rows, A.nnz, 0, Ac.dtype)
    ws = torch.empty(max(ws_b, 256), dtype=torch.uint8, device=dev)
    ev_x = [torch.cuda.Event() for _ in range(2)]
    ev_c = [torch.cuda.Event() for _ in range(2)]
    ev_o = [torch.cuda.Event() for _ in range(2)]
    for e in ev_c + ev_o:
        e.record(torch.cuda.current_stream(dev))

    def step(i):
        b = i % 2
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_c[b])            # x buffer b free (SpMV i-2 done)
            d_x[b].copy_(h_x[b], non_blocking=True)
            ev_x[b].record(s_in)
        s_comp.wait_event(ev_x[b])
        s_comp.wait_event(ev_o[b])              # y buffer b free (download i-2 done)
        if hx is not None:
            _lib.check(lib.lw_spmv_work_oriented_hotx(Hc, hot_ptr, hx.n_hot, d_x[b].data_ptr(),
                                                      d_y[b].data_ptr(), 0, ws.data_ptr(), ws.numel(),
                                                      int(s_comp.cuda_stream)), "lw_spmv_work_oriented_hotx")
        else:
            _lib.check(lib.lw_spmv(_lib.LW_MERGE_PATH, Ac, d_x[b].data_ptr(), d_y[b].data_ptr(), 0, 32,
                                   32, ws.data_ptr(), ws.numel(), int(s_comp.cuda_stream)), "lw_spmv")
        ev_c[b].record(s_comp)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_c[b])
            h_y[b].copy_(d_y[b], non_blocking=True)
            ev_o[b].record(s_out)

    for i in range(4):
        step(i)
    torch.cuda.synchronize()
    # a serving loop's steady state: the pipeline's fill (first upload) and drain
    # (last SpMV + download), ~2.2 ms in all, are spread over >= 100 steps
    steps = max(args.steps, 100)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(s_in)
    s_comp.wait_event(t0)
    s_out.wait_event(t0)
    for i in range(steps):
        step(i)
    s_out.wait_event(ev_c[(steps - 1) % 2])
    t1.record(s_out)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    # the PCIe ceiling of the same copies with no SpMV: x up and y down at once
    c0 = torch.cuda.Event(enable_timing=True)
    c1 = torch.cuda.Event(enable_timing=True)
    c0.record(s_in)
    s_out.wait_event(c0)
    for i in range(10):
        with torch.cuda.stream(s_in):
            d_x[i % 2].copy_(h_x[i % 2], non_blocking=True)
        with torch.cuda.stream(s_out):
            h_y[i % 2].copy_(d_y[i % 2], non_blocking=True)
    s_out.wait_stream(s_in)
    c1.record(s_out)
    torch.cuda.synchronize()
    copy_ms = c0.elapsed_time(c1) / 10
    return {"value": round(2.0 * nnz_total / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(h_x[0].numel() * h_x[0].element_size()),
            "d2h_bytes_per_step": int(h_y[0].numel() * h_y[0].element_size()),
            "ms_per_step": round(ms, 3), "steps": steps,
            "copies_only_ms_per_step": round(copy_ms, 3),
            "path": (("lw_spmv_work_oriented_hotx" if hx is not None else "lw_spmv") +
                     " (C ABI) per step; pinned host x copied in and y copied out every "
                     "step on separate streams, double-buffered so uploads/downloads overlap "
                     "the neighbouring steps' SpMV; matrix resident in HBM (uploaded once, "
                     "outside the timed region)")}


def e2e_host(A, args, lib, dev, nnz_total):
    import torch

    from paper_2301_04792_b200 import _lib

    h_off = A.row_offsets.cpu().pin_memory()
    h_col = A.col_indices.cpu().pin_memory()
    h_val = A.values.cpu().pin_memory()
    h_x = torch.ones(A.cols, dtype=A.dtype).pin_memory()
    h_y = torch.empty(A.rows, dtype=A.dtype).pin_memory()
    H = _lib.LwCsr()
    H.rows, H.cols, H.nnz = A.rows, A.cols, A.nnz
    H.row_offsets, H.col_indices, H.values = h_off.data_ptr(), h_col.data_ptr(), h_val.data_ptr()
    H.offset_bits, H.dtype = A.offset_bits, A.c_struct().dtype
    stream = torch.cuda.current_stream(dev)
    sp = int(stream.cuda_stream)
    steps = max(2, min(args.steps, 5))
    for _ in range(2):
        _lib.check(lib.lw_spmv_host(_lib.LW_MERGE_PATH, H, h_x.data_ptr(), h_y.data_ptr(), 0, 32,
                                    32, sp), "lw_spmv_host")
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        _lib.check(lib.lw_spmv_host(_lib.LW_MERGE_PATH, H, h_x.data_ptr(), h_y.data_ptr(), 0, 32,
                                    32, sp), "lw_spmv_host")
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    h2d = (h_off.numel() * h_off.element_size() + h_col.numel() * 4
           + h_val.numel() * h_val.element_size() + h_x.numel() * h_x.element_size())
    return {"value": round(2.0 * nnz_total / (ms * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(h_y.numel() * h_y.element_size()),
            "ms_per_step": round(ms, 3), "steps": steps,
            "path": "lw_spmv_host (C ABI, pinned host CSR + x in, y out, stream-synchronized)"}


def host_cpu() -> dict:
    """The host the CPU legs ran on: lscpu model name, logical CPUs usable here."""
    model = None
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    cpus = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    return {"model": model, "logical_cpus": cpus}


def cpu_baseline(A, args):
    """Reference CPU algorithm (oracle port of lanework merge-path, fp64) on the
    same matrix, all host threads (lanes = 32 x threads, the reference CLI's
    configuration) and 1 thread (32 lanes, the reference's default config);
    median of --cpu-reps runs, the reference CLI's protocol (cli.py:137-145)."""
    from oracle import oracle

    threads = oracle.default_threads()
    off = A.row_offsets.cpu().numpy().astype(np.int64)
    col = A.col_indices.cpu().numpy().astype(np.int64)
    val = A.values.cpu().numpy().astype(np.float64)
    x = np.ones(A.cols)

    def med(th, reps):
        oracle.spmv(off, col, val, x, "merge-path", lanes=32 * th, threads=th)
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            oracle.spmv(off, col, val, x, "merge-path", lanes=32 * th, threads=th)
            ts.append(time.perf_counter() - t)
        return float(np.median(ts))

    sec = med(threads, max(args.cpu_reps, 3))
    sec1 = med(1, 1)
    return {"value": round(2.0 * A.nnz / sec / 1e9, 4), "unit": "GFLOP/s", "cores": threads,
            "kind": "port", "ms_per_step": round(sec * 1e3, 2),
            "one_thread": {"value": round(2.0 * A.nnz / sec1 / 1e9, 4), "ms_per_step": round(sec1 * 1e3, 1),
                           "lanes": 32},
            "host": host_cpu(),
            "sample": (f"full matrix ({A.rows} rows, {A.nnz} nnz), oracle port of lanework "
                       f"merge-path (fp64/int64), {32 * threads} lanes on {threads} threads, median of "
                       f"{max(args.cpu_reps, 3)}; one_thread: 32 lanes on 1 thread, 1 run")}


def _free_port() -> int:
    import socket

    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int | None:
    """`python bench.py --gpus N` (N > 1) outside torchrun re-executes itself
    under torch.distributed.run with N ranks on this node (127.0.0.1
    rendezvous), so the driver's plain command and its torchrun form give the
    same N-rank run. NCCL's INIT log stays on (the driver counts ranks from it);
    rank 0 prints the JSON line after the communicators are destroyed, so it is
    the last line of stdout. Returns the child's exit code, or None when this
    process is already a rank (or N == 1, or the reference arm: rank 0 only)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return None
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def check_world(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl != "reference" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} "
                         f"(launch with --nproc-per-node {args.gpus}, or without torchrun)")


def dry_run(args) -> None:
    """--dry-run: the launch path alone (rendezvous, one all-reduce over gloo,
    the rank count on rank 0's line) — no device work; CPU-testable."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    seen = world
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        seen = int(t.item())
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_in_allreduce": seen}), flush=True)


def main():
    args = parse()
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    check_world(args)
    if args.dry_run:
        dry_run(args)
    elif args.impl == "reference":
        reference_arm(args)
    elif args.mode == "power":
        power_arm(args)
    else:
        our_arm(args)


if __name__ == "__main__":
    main()
