"""Executor configuration, imbalance accounting and host schedule walkers.

``ExecutorConfig`` keeps the reference's fields, defaults and validation
(executor.py:35-72): ``lanes=None`` resolves to ``worker_threads*32`` in
``__post_init__``, so reference code that reads ``cfg.lanes`` (or passes the
config to ``imbalance`` and the walkers) sees exactly the reference's number.
What the GPU launch does with it is recorded separately: a config built
without an explicit ``lanes`` carries ``lanes_auto=True`` and the cuda backend
then sizes P for the device (``lw_auto_lanes``, one resident wave of each
kernel) instead of launching the reference's 32 CPU lanes, which would leave a
B200 idle; an explicit ``lanes=P`` is launched as P lanes. ``device_config``
returns the config with the launch's lane count filled in, so
``imbalance(ts, device_config(cfg, m))`` predicts the per-thread atom counts of
the actual launch.

``execute_tile_major`` / ``execute_merge_path`` / ``fixup_combine`` are the
reference's callback API for custom per-atom work (executor.py:132-221). They
walk the same Schedule objects on the host (Python callbacks cannot run on the
GPU) and are not on the SpMV path.
"""

from __future__ import annotations

import operator
import threading
from dataclasses import dataclass, field, replace
from typing import Callable, NamedTuple

import numpy as np

from .schedules import (GroupMappedSchedule, MergePathSchedule, ScheduleKind,
                        ThreadMappedSchedule, merge_path_partition, num_blocks)
from .work import tile_offsets

__all__ = ["AtomicMinArray", "atomic_min_real", "SENTINEL_TILE", "ExecutorConfig", "CarryOut", "CarryPolicy", "SUM_CARRIES",
           "ImbalanceReport", "imbalance", "execute_tile_major", "execute_merge_path",
           "fixup_combine", "device_config"]

SENTINEL_TILE = -1


@dataclass
class ExecutorConfig:
    """Lane count P, the schedule mapping lanes to work, and group shape."""

    schedule: ScheduleKind = ScheduleKind.MERGE_PATH
    lanes: int | None = None
    worker_threads: int = 1
    group_size: int = 32
    tiles_per_block: int | None = None
    # True when lanes was not given: the device launch is sized for the GPU.
    # Not an __init__ argument, so dataclasses.replace(cfg, lanes=P) is explicit.
    lanes_auto: bool = field(default=False, init=False, repr=False, compare=False)

    def __post_init__(self):
        if not isinstance(self.schedule, ScheduleKind):
            self.schedule = ScheduleKind(self.schedule)
        if self.worker_threads < 1:
            raise ValueError("worker_threads must be >= 1")
        if self.lanes is None:
            self.lanes = self.worker_threads * 32
            self.lanes_auto = True
        if self.lanes < 1:
            raise ValueError("lanes must be >= 1")
        if self.group_size < 1:
            raise ValueError("group_size must be >= 1")
        if self.tiles_per_block is None:
            self.tiles_per_block = self.group_size
        if self.tiles_per_block < 1:
            raise ValueError("tiles_per_block must be >= 1")

    @property
    def lane_count(self) -> int:
        """Lanes for host-side accounting (== lanes, the reference's P)."""
        return self.lanes

    def group_lanes(self, group_id: int) -> range:
        lo = group_id * self.group_size
        return range(lo, min(lo + self.group_size, self.lane_count))

    @property
    def group_count(self) -> int:
        return (self.lane_count + self.group_size - 1) // self.group_size


def device_config(cfg: ExecutorConfig, m) -> ExecutorConfig:
    """``cfg`` with ``lanes`` fixed to the value the device kernels will use for ``m``."""
    if not cfg.lanes_auto:
        return cfg
    from . import _lib

    code = {ScheduleKind.THREAD_MAPPED: _lib.LW_THREAD_MAPPED,
            ScheduleKind.MERGE_PATH: _lib.LW_MERGE_PATH,
            ScheduleKind.GROUP_MAPPED: _lib.LW_GROUP_MAPPED}[cfg.schedule]
    lanes = _lib.auto_lanes(code, int(m.rows), int(m.nnz), cfg.group_size, cfg.tiles_per_block)
    return replace(cfg, lanes=lanes)


class CarryOut(NamedTuple):
    """Partial reduction of a lane's right-open trailing tile (or the sentinel)."""

    tile: int
    partial: float


@dataclass(frozen=True)
class CarryPolicy:
    identity: float = 0.0
    combine: Callable = operator.add


SUM_CARRIES = CarryPolicy()


@dataclass
class ImbalanceReport:
    per_lane_atoms: np.ndarray
    max: int = field(init=False)
    mean: float = field(init=False)
    imbalance_factor: float = field(init=False)

    def __post_init__(self):
        a = self.per_lane_atoms
        self.max = int(a.max()) if a.size else 0
        self.mean = float(a.mean()) if a.size else 0.0
        self.imbalance_factor = self.max / self.mean if self.mean > 0 else 1.0


def imbalance(ts, cfg: ExecutorConfig) -> ImbalanceReport:
    """Atoms per lane under ``cfg`` without running anything (executor.py:224-251)."""
    p = cfg.lane_count
    lengths = np.diff(tile_offsets(ts)).astype(np.int64)
    out = np.zeros(p, dtype=np.int64)
    kind = cfg.schedule
    if kind is ScheduleKind.THREAD_MAPPED:
        n = lengths.size
        if n:
            pad = (-n) % p
            out[:] = np.concatenate([lengths, np.zeros(pad, np.int64)]).reshape(-1, p).sum(axis=0)
    elif kind is ScheduleKind.MERGE_PATH:
        c = merge_path_partition(ts, p)
        out[:] = np.diff(c[:, 1])
    elif kind is ScheduleKind.GROUP_MAPPED:
        off = tile_offsets(ts)
        tpb, gs, groups = cfg.tiles_per_block, cfg.group_size, cfg.group_count
        n_t = ts.num_tiles
        for b in range(num_blocks(ts, tpb)):
            gid = b % groups
            total = int(off[min((b + 1) * tpb, n_t)] - off[b * tpb])
            lo = gid * gs
            members = min(gs, p - lo)
            if members <= 0 or total == 0:
                continue
            m = np.arange(members)
            out[lo:lo + members] += np.maximum(0, (total - m + members - 1) // members)
    else:  # pragma: no cover
        raise ValueError(f"unknown schedule {kind}")
    return ImbalanceReport(out)


def _schedule_for(ts, cfg: ExecutorConfig):
    if cfg.schedule is ScheduleKind.THREAD_MAPPED:
        return ThreadMappedSchedule(ts, cfg.lane_count)
    if cfg.schedule is ScheduleKind.GROUP_MAPPED:
        return GroupMappedSchedule(ts, cfg.lane_count, cfg.group_size, cfg.tiles_per_block)
    return MergePathSchedule(ts, cfg.lane_count)


def execute_tile_major(cfg: ExecutorConfig, ts, work_fn) -> None:
    """Call ``work_fn(lane, tile, atom_range)`` over the tile set (executor.py:132-170).

    Thread-mapped lanes see each owned tile once with its whole atom range;
    group-mapped members see their block atoms one at a time in member-stride
    order, attributed to the tile the block plan assigns.
    """
    if cfg.schedule is ScheduleKind.MERGE_PATH:
        raise ValueError(f"execute_tile_major does not accept {cfg.schedule}")
    sched = _schedule_for(ts, cfg)
    if cfg.schedule is ScheduleKind.THREAD_MAPPED:
        for lane in range(sched.lanes):
            for tile in sched.tiles(lane):
                work_fn(lane, tile, sched.atoms(lane, tile))
        return
    off = sched.offsets
    tpb, n_t = sched.tiles_per_block, ts.num_tiles
    for gid in range(sched.group_count):
        lanes = cfg.group_lanes(gid)
        members = len(lanes)
        if members == 0:
            continue
        for b in range(gid, num_blocks(ts, tpb), sched.group_count):
            first, last = b * tpb, min((b + 1) * tpb, n_t)
            base = int(off[first])
            total = int(off[last]) - base
            for m, lane in enumerate(lanes):
                tile = first
                for local in range(m, total, members):
                    atom = base + local
                    while int(off[tile + 1]) <= atom:
                        tile += 1
                    work_fn(lane, tile, range(atom, atom + 1))


def execute_merge_path(cfg: ExecutorConfig, ts, atom_fn, tile_done,
                       carry_policy: CarryPolicy = SUM_CARRIES) -> list[CarryOut]:
    """Walk every merge-path slice in path order (executor.py:173-209).

    ``tile_done(lane, tile, acc)`` fires for tiles whose right edge lies in the
    slice; a trailing right-open tile comes back as the lane's CarryOut.
    """
    if cfg.schedule is not ScheduleKind.MERGE_PATH:
        raise ValueError(f"execute_merge_path requires the merge-path schedule, got {cfg.schedule}")
    sched = MergePathSchedule(ts, cfg.lane_count)
    off = sched.offsets
    ident, comb = carry_policy.identity, carry_policy.combine
    carries = [CarryOut(SENTINEL_TILE, ident)] * sched.lanes
    for lane in range(sched.lanes):
        s = sched.slice(lane)
        atom = s.atom_begin
        for tile in range(s.tile_begin, s.tile_end):
            acc = ident
            stop = int(off[tile + 1])
            while atom < stop:
                acc = comb(acc, atom_fn(lane, tile, atom))
                atom += 1
            tile_done(lane, tile, acc)
        if atom < s.atom_end:
            acc = ident
            while atom < s.atom_end:
                acc = comb(acc, atom_fn(lane, s.tile_end, atom))
                atom += 1
            carries[lane] = CarryOut(s.tile_end, acc)
    return carries


def fixup_combine(carries, combine) -> None:
    """Apply every non-sentinel carry once, in lane order (executor.py:212-221)."""
    for c in carries:
        if c.tile != SENTINEL_TILE:
            combine(c.tile, c.partial)


class AtomicMinArray:
    """Slots of non-negative reals (or +inf) with an atomic min — the host twin
    of the device kernels' relaxation (csrc/frontier.cu), built the same way:
    a non-negative double orders exactly like its 64-bit pattern read as a
    signed integer, so the min is an integer compare-and-store on the bits.
    Python has no CAS, so each store runs under one of a fixed set of striped
    locks (slot i uses lock i % STRIPES): updates of one slot are serialised,
    updates of different slots mostly are not. Negative values are rejected
    (their bit patterns would order backwards), as in reference
    executor.py:254-283."""

    STRIPES = 64

    def __init__(self, values: np.ndarray):
        vals = np.asarray(values, dtype=np.float64)
        if vals.size and bool((vals < 0).any()):
            raise ValueError("slots must hold non-negative reals or +inf")
        self.values = vals
        self._bits = vals.view(np.int64)
        self._locks = tuple(threading.Lock() for _ in range(self.STRIPES))

    def atomic_min(self, index: int, candidate: float) -> float:
        """Lower slot ``index`` to ``candidate`` if smaller; returns the prior value."""
        c = float(candidate)
        if not c >= 0.0:
            raise ValueError("candidate must be non-negative")
        bits = int(np.float64(c + 0.0).view(np.int64))   # + 0.0 folds -0.0 into +0.0
        with self._locks[index % self.STRIPES]:
            prior = int(self._bits[index])
            if bits < prior:
                self._bits[index] = bits
        return float(np.int64(prior).view(np.float64))


def atomic_min_real(slots: AtomicMinArray, index: int, candidate: float) -> float:
    """Function form of :meth:`AtomicMinArray.atomic_min`."""
    return slots.atomic_min(index, candidate)
