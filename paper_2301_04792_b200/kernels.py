"""The SpMV operator on the cuda backend (reference kernels.py:57-126, 211-227).

``spmv(m, x, cfg)`` keeps the reference signature and error behaviour:
  * host operands (CsrMatrix + NumPy x): x is validated exactly like
    kernels.py:60-62 (ValueError on a length mismatch), x is uploaded (the
    matrix once: its device copy is cached on the CsrMatrix while its arrays
    are unchanged, see device.cached_device_csr), the schedule's kernel runs,
    and a NumPy float64 y comes back — computed in fp64 on the device by
    default, the reference's precision;
  * device operands (DeviceCsr + torch CUDA x): y stays on the device in the
    matrix's dtype; nothing touches the host. This is the path the bench's
    ``value`` measures.
Schedule selection follows ``cfg.schedule``; a config built without ``lanes``
(``cfg.lanes_auto``) lets the device size the lane count (see
executor.device_config); an explicit ``lanes=P`` launches P lanes.
"""

from __future__ import annotations

import functools
from dataclasses import dataclass, replace

import numpy as np

from . import _backend, _lib
from .device import (DeviceCsr, Probe, Workspace, cached_device_csr, current_stream, device_to_host,
                     host_to_device)
from .executor import ExecutorConfig
from .schedules import ScheduleKind

__all__ = ["spmv", "spmm", "spmv_probe", "spmv_auto", "choose_spmv_schedule",
           "HeuristicConfig", "schedule_code"]

_WS = Workspace()


def schedule_code(kind: ScheduleKind) -> int:
    return {ScheduleKind.THREAD_MAPPED: _lib.LW_THREAD_MAPPED,
            ScheduleKind.MERGE_PATH: _lib.LW_MERGE_PATH,
            ScheduleKind.GROUP_MAPPED: _lib.LW_GROUP_MAPPED}[kind]


def _lanes_arg(cfg: ExecutorConfig) -> int:
    return 0 if cfg.lanes_auto else int(cfg.lanes)


@functools.lru_cache(maxsize=256)
def _wo_workspace(rows: int, nnz: int, lanes: int, dtype_code: int) -> int:
    return _lib.load().lw_spmv_work_oriented_workspace(rows, nnz, lanes, dtype_code)


@functools.lru_cache(maxsize=256)
def _hotx_workspace(rows: int, nnz: int, lanes: int, n_hot: int, dtype_code: int) -> int:
    return _lib.load().lw_spmv_work_oriented_hotx_workspace(rows, nnz, lanes, n_hot, dtype_code)


@functools.lru_cache(maxsize=256)
def _mm_workspace(code: int, rows: int, nnz: int, n: int, lanes: int, dtype_code: int) -> int:
    return _lib.load().lw_spmm_workspace(code, rows, nnz, n, lanes, dtype_code)


def _launch(m: DeviceCsr, x, y, cfg: ExecutorConfig, probe: Probe | None, stream: int) -> None:
    lib = _lib.load()
    A = m.c_struct()
    xp = x.data_ptr() if x.numel() else None
    yp = y.data_ptr() if y.numel() else None
    pp = probe.c_struct() if probe is not None else None
    lanes = _lanes_arg(cfg)
    kind = cfg.schedule
    if kind is ScheduleKind.THREAD_MAPPED:
        rc = lib.lw_spmv_thread_mapped(A, xp, yp, lanes, pp, stream)
    elif kind is ScheduleKind.MERGE_PATH and probe is None and (hx := m.hot_columns()) is not None:
        need = _hotx_workspace(m.rows, m.nnz, lanes, hx.n_hot, A.dtype)
        ws = _WS.get(need, m.device, stream)
        rc = lib.lw_spmv_work_oriented_hotx(hx.packed.c_struct(), hx.hot_cols.data_ptr() if hx.n_hot else None,
                                            hx.n_hot, xp, yp, lanes, ws.data_ptr(), ws.numel(), stream)
    elif kind is ScheduleKind.MERGE_PATH:
        need = _wo_workspace(m.rows, m.nnz, lanes, A.dtype)
        ws = _WS.get(need, m.device, stream)
        rc = lib.lw_spmv_work_oriented(A, xp, yp, lanes, ws.data_ptr(), ws.numel(), pp, stream)
    else:
        rc = lib.lw_spmv_group_mapped(A, xp, yp, lanes, cfg.group_size, cfg.tiles_per_block, pp,
                                      stream)
    _lib.check(rc, f"spmv[{kind.value}]")


def _check_device_x(m: DeviceCsr, x):
    import torch

    if not isinstance(x, torch.Tensor):
        raise TypeError("a DeviceCsr needs x as a torch CUDA tensor")
    if x.ndim != 1 or x.shape[0] != m.cols:
        raise ValueError(f"x has length {x.numel()}, expected {m.cols}")
    if x.device != m.device:
        raise ValueError(f"x is on {x.device}, matrix on {m.device}")
    if x.dtype != m.dtype:
        raise ValueError(f"x dtype {x.dtype} differs from matrix dtype {m.dtype}")
    return x.contiguous()


def spmv(m, x, cfg: ExecutorConfig | None = None, *, out=None, dtype=None):
    """y = m @ x under ``cfg.schedule``; rows without nonzeros yield 0."""
    cfg = cfg or ExecutorConfig()
    _backend.require_cuda()
    import torch

    if isinstance(m, DeviceCsr):
        x = _check_device_x(m, x)
        y = out if out is not None else torch.empty(m.rows, dtype=m.dtype, device=m.device)
        if (y.shape != (m.rows,) or y.dtype != m.dtype or y.device != m.device
                or not y.is_contiguous()):
            raise ValueError("out must be a contiguous vector of length rows with the matrix dtype")
        _launch(m, x, y, cfg, None, current_stream(m.device))
        return y
    xh = np.ascontiguousarray(x, dtype=np.float64)
    if xh.ndim != 1 or xh.size != m.cols:
        raise ValueError(f"x has length {xh.size}, expected {m.cols}")
    dm = cached_device_csr(m, dtype=dtype or "float64")
    xd = host_to_device(xh, dm.device, dm.dtype)
    if (cfg.schedule in _OVERLAP_SCHEDULES and cfg.lanes_auto and dm.dtype == torch.float64
            and dm.nnz >= _OVERLAP_MIN_NNZ):
        return _spmv_host_overlapped(dm, m.row_offsets, xd, cfg)
    y = torch.empty(dm.rows, dtype=dm.dtype, device=dm.device)
    _launch(dm, xd, y, cfg, None, current_stream(dm.device))
    return device_to_host(y.to(torch.float64))


# Host-operand SpMV on large matrices: y goes down in row blocks, each block's
# download overlapping the SpMV of the blocks after it (C3 fp64: the 128 MB y
# download took 2.4 ms after a 1.5 ms SpMV). The download is the longer of the
# two, so it should start early and never wait: the blocks have equal rows (equal
# download time) and run lightest first (fewest merge-path items = rows + atoms),
# so the first download starts after the cheapest SpMV and every later block's
# SpMV fits under the download before it. Only for the device-sized lane count,
# and for the schedules whose row sums do not depend on where a launch starts:
# thread_mapped (a row's atoms in order on one thread: y bit-identical) and
# merge-path (each block is its own partition, so rows a lane boundary cuts may
# add their partials in a different grouping than one whole-matrix launch: fp64,
# far inside the 1e-12 bound; integer data stay bit-exact). group_mapped keeps
# one launch: its member-major steps are aligned to each group's first atom.
_OVERLAP_MIN_NNZ = 1 << 22
_OVERLAP_SCHEDULES = (ScheduleKind.MERGE_PATH, ScheduleKind.THREAD_MAPPED)
_OVERLAP_BLOCKS = 8
_COPY_STREAMS = {}


def _row_blocks(dm: DeviceCsr, host_offsets, parts: int):
    """(Nearly) equal-row blocks [(r0, r1, DeviceCsr view)] in increasing order of
    their merge-path items, cached on the DeviceCsr while its tensors are unchanged."""
    from .device import _same_key

    key = dm._tensor_key()
    hit = dm.__dict__.get("_lw_row_blocks")
    if hit is not None and hit[0] == parts and _same_key(hit[1], key):
        return hit[2]
    off = np.asarray(host_offsets, dtype=np.int64)
    bounds = np.linspace(0, dm.rows, parts + 1).astype(np.int64)
    # move each inner bound to the next row whose first atom is 8-aligned, so every
    # block's col_idx / values start on a 32-byte boundary (the kernels' vector
    # loads need it; thread_mapped then also keeps its two chains bit-identical)
    for i in range(1, parts):
        near = off[bounds[i]: min(bounds[i] + 4096, dm.rows)]
        hit = np.flatnonzero(near % 8 == 0)
        if hit.size:
            bounds[i] += hit[0]
    bounds = np.unique(np.maximum.accumulate(bounds))
    items = (bounds[1:] - bounds[:-1]) + (off[bounds[1:]] - off[bounds[:-1]])
    blocks = [(int(bounds[i]), int(bounds[i + 1]), dm.row_slice(int(bounds[i]), int(bounds[i + 1])))
              for i in np.argsort(items, kind="stable")]
    dm.__dict__["_lw_row_blocks"] = (parts, key, blocks)
    return blocks


def _spmv_host_overlapped(dm: DeviceCsr, host_offsets, xd, cfg: ExecutorConfig):
    import torch

    stream = torch.cuda.current_stream(dm.device)
    copy = _COPY_STREAMS.get(dm.device)
    if copy is None:
        copy = _COPY_STREAMS[dm.device] = torch.cuda.Stream(dm.device)
    y = torch.empty(dm.rows, dtype=torch.float64, device=dm.device)
    yh = torch.empty(dm.rows, dtype=torch.float64, pin_memory=True)
    for r0, r1, blk in _row_blocks(dm, host_offsets, _OVERLAP_BLOCKS):
        _launch(blk, xd, y[r0:r1], cfg, None, stream.cuda_stream)
        ev = torch.cuda.Event()
        ev.record(stream)
        copy.wait_event(ev)
        with torch.cuda.stream(copy):
            yh[r0:r1].copy_(y[r0:r1], non_blocking=True)
    y.record_stream(copy)
    copy.synchronize()
    return yh.numpy()


def _launch_spmm(m: DeviceCsr, B, C, cfg: ExecutorConfig, stream: int) -> None:
    lib = _lib.load()
    A = m.c_struct()
    n = int(B.shape[1])
    code = schedule_code(cfg.schedule)
    lanes = _lanes_arg(cfg)
    bp = B.data_ptr() if B.numel() else None
    cp = C.data_ptr() if C.numel() else None
    need = _mm_workspace(code, m.rows, m.nnz, n, lanes, A.dtype)
    ws = _WS.get(need, m.device, stream) if need else None
    rc = lib.lw_spmm(code, A, bp, cp, n, lanes, cfg.group_size, cfg.tiles_per_block,
                     ws.data_ptr() if ws is not None else None, need, stream)
    _lib.check(rc, f"spmm[{cfg.schedule.value}]")


def spmm(m, B, cfg: ExecutorConfig | None = None, *, out=None, dtype=None):
    """C = m @ B for a dense row-major B (reference kernels.py:129-175).

    Host operands (CsrMatrix + array-like B): B is validated like the reference
    (2-D with B.shape[0] == m.cols, else ValueError), computed on the device in
    fp64 by default and returned as a NumPy float64 [rows, k] array. Device
    operands (DeviceCsr + torch CUDA B [cols, k] in the matrix dtype): C stays on
    the device. The schedule assigns tiles and atoms to lanes exactly as spmv does.
    """
    cfg = cfg or ExecutorConfig()
    _backend.require_cuda()
    import torch

    if isinstance(m, DeviceCsr):
        if not isinstance(B, torch.Tensor):
            raise TypeError("a DeviceCsr needs B as a torch CUDA tensor")
        if B.ndim != 2 or B.shape[0] != m.cols:
            raise ValueError(f"B has shape {tuple(B.shape)}, expected ({m.cols}, k)")
        if B.device != m.device or B.dtype != m.dtype:
            raise ValueError("B must be on the matrix's device with the matrix dtype")
        B = B.contiguous()
        C = out if out is not None else torch.empty((m.rows, B.shape[1]), dtype=m.dtype,
                                                    device=m.device)
        if (C.shape != (m.rows, B.shape[1]) or C.dtype != m.dtype or C.device != m.device
                or not C.is_contiguous()):
            raise ValueError("out must be a contiguous [rows, k] tensor with the matrix dtype")
        _launch_spmm(m, B, C, cfg, current_stream(m.device))
        return C
    Bh = np.ascontiguousarray(B, dtype=np.float64)
    if Bh.ndim != 2 or Bh.shape[0] != m.cols:
        raise ValueError(f"B has shape {Bh.shape}, expected ({m.cols}, k)")
    dm = cached_device_csr(m, dtype=dtype or "float64")
    Bd = host_to_device(Bh, dm.device, dm.dtype)
    C = torch.empty((dm.rows, Bh.shape[1]), dtype=dm.dtype, device=dm.device)
    _launch_spmm(dm, Bd, C, cfg, current_stream(dm.device))
    return device_to_host(C.to(torch.float64))


def spmv_probe(m: DeviceCsr, x, cfg: ExecutorConfig | None = None):
    """Instrumented SpMV: returns (y, probe dict, lanes) for bit-exact schedule checks.

    probe["lane_atoms"][l] is the atoms lane l processed; probe["atom_lane"][a] /
    ["atom_tile"][a] the lane and tile atom a was processed by / attributed to;
    probe["atom_visits"][a] how often it was processed (must be 1).
    """
    from .executor import device_config

    cfg = device_config(cfg or ExecutorConfig(), m)
    _backend.require_cuda()
    import torch

    x = _check_device_x(m, x)
    y = torch.empty(m.rows, dtype=m.dtype, device=m.device)
    probe = Probe(cfg.lanes, m.nnz, m.device)
    _launch(m, x, y, cfg, probe, current_stream(m.device))
    return y, probe.host(), cfg.lanes


@dataclass(frozen=True)
class HeuristicConfig:
    """Size thresholds of the schedule dispatcher (alpha=500, beta=10000)."""

    alpha: int = 500
    beta: int = 10000

    def __post_init__(self):
        if self.alpha <= 0 or self.beta <= 0:
            raise ValueError("alpha and beta must be positive")


def choose_spmv_schedule(rows: int, cols: int, nnz: int, heuristic: HeuristicConfig | None = None,
                         small_schedule: ScheduleKind = ScheduleKind.THREAD_MAPPED) -> ScheduleKind:
    """Merge-path unless the matrix is small in a dimension and in nnz (kernels.py:211-218)."""
    h = heuristic or HeuristicConfig()
    small = (rows < h.alpha or cols < h.alpha) and nnz < h.beta
    return small_schedule if small else ScheduleKind.MERGE_PATH


def spmv_auto(m, x, heuristic: HeuristicConfig | None = None, cfg: ExecutorConfig | None = None,
              small_schedule: ScheduleKind = ScheduleKind.THREAD_MAPPED):
    """SpMV under the heuristic's schedule; returns (y, chosen) (kernels.py:221-227)."""
    chosen = choose_spmv_schedule(m.rows, m.cols, m.nnz, heuristic, small_schedule)
    cfg = replace(cfg, schedule=chosen) if cfg is not None else ExecutorConfig(schedule=chosen)
    return spmv(m, x, cfg), chosen
