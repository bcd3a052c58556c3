"""Schedules: maps from lane ids to tiles and atoms.

Host-side API with the reference's names and return types (schedules.py:21-167):
``ScheduleKind``, ``thread_mapped_tiles``, ``merge_path_search``,
``merge_path_partition``, ``merge_path_slices``, ``exclusive_prefix_sum``,
``group_plan``, ``get_tile``. The device kernels implement the same maps with
one lane per GPU thread (see csrc/); ``merge_path_partition(ts, P,
device=...)`` runs the device search (lw_merge_path_partition) and is bit-exact
with the host result.

``Schedule`` objects add the range-based iteration the paper's listings use
(PAPER.md:273-288): ``schedule.tiles(lane)`` and ``schedule.atoms(lane, tile)``.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from .work import lane_stride_range, tile_offsets

__all__ = [
    "ScheduleKind", "MergePathCoord", "MergePathSlice", "GroupPlan", "thread_mapped_tiles",
    "merge_path_search", "merge_path_partition", "merge_path_slices", "exclusive_prefix_sum",
    "num_blocks", "group_plan", "get_tile", "Schedule", "ThreadMappedSchedule",
    "MergePathSchedule", "GroupMappedSchedule", "make_schedule",
]


class ScheduleKind(enum.Enum):
    """Schedule names; values are the reference's CLI names (schedules.py:21-24).

    ``WORK_ORIENTED`` is the north star's name for the merge-path schedule and is
    an alias of ``MERGE_PATH``; "work-oriented"/"work_oriented" parse to it.
    """

    THREAD_MAPPED = "thread-mapped"
    MERGE_PATH = "merge-path"
    GROUP_MAPPED = "group-mapped"
    WORK_ORIENTED = "merge-path"  # alias

    @classmethod
    def _missing_(cls, value):
        if isinstance(value, str):
            key = value.strip().lower().replace("_", "-")
            aliases = {"work-oriented": cls.MERGE_PATH, "merge": cls.MERGE_PATH,
                       "thread": cls.THREAD_MAPPED, "group": cls.GROUP_MAPPED,
                       "warp-mapped": cls.GROUP_MAPPED, "block-mapped": cls.GROUP_MAPPED}
            for member in cls:
                if member.value == key:
                    return member
            return aliases.get(key)
        return None


class MergePathCoord(NamedTuple):
    tile: int
    atom: int


class MergePathSlice(NamedTuple):
    tile_begin: int
    atom_begin: int
    tile_end: int
    atom_end: int

    @property
    def work_items(self) -> int:
        return (self.tile_end - self.tile_begin) + (self.atom_end - self.atom_begin)


@dataclass
class GroupPlan:
    """A tile block and the exclusive prefix sum of its tiles' atom counts."""

    tile_begin: int
    tile_count: int
    prefix: np.ndarray

    @property
    def total_atoms(self) -> int:
        return int(self.prefix[-1])


def thread_mapped_tiles(ts, lane: int, lane_count: int) -> range:
    """Tiles of ``lane`` under thread-mapped: lane, lane+P, ...."""
    return lane_stride_range(lane, lane_count, ts.num_tiles)


def merge_path_search(diagonal: int, ts) -> MergePathCoord:
    """Coordinate of the merge path on ``diagonal`` (reference schedules.py:63-85).

    The path consumes a tile boundary once all of the tile's atoms are consumed,
    boundaries winning ties (so an empty tile costs one step). The point on
    diagonal d is (t, d-t) for the largest feasible t with offsets[t] <= d - t.
    """
    n_t, n_a = ts.num_tiles, ts.num_atoms
    if diagonal < 0 or diagonal > n_t + n_a:
        raise ValueError(f"diagonal {diagonal} outside [0, {n_t + n_a}]")
    off = tile_offsets(ts)
    lo, hi = max(0, diagonal - n_a), min(diagonal, n_t)
    while hi > lo:
        probe = (lo + hi + 1) >> 1
        if int(off[probe]) + probe <= diagonal:
            lo = probe
        else:
            hi = probe - 1
    return MergePathCoord(lo, diagonal - lo)


def _partition_diagonals(total: int, lane_count: int) -> np.ndarray:
    quota = (total + lane_count - 1) // lane_count if total else 0
    return np.minimum(np.arange(lane_count + 1, dtype=np.int64) * quota, total)


def merge_path_partition(ts, lane_count: int, device=None) -> np.ndarray:
    """``(lane_count+1, 2)`` int64 split points (tile, atom) of the merge path.

    Every lane gets ``ceil(total/lane_count)`` items except where the clamp at
    ``total`` bites (reference schedules.py:88-110). With ``device`` set (a torch
    device or DeviceCsr) the search runs on the GPU through
    ``lw_merge_path_partition`` and a torch int64 tensor is returned.
    """
    if lane_count < 1:
        raise ValueError("lane_count must be >= 1")
    if device is not None:
        from .device import device_merge_path_partition

        return device_merge_path_partition(ts, lane_count, device)
    off = tile_offsets(ts)
    n_t = ts.num_tiles
    diag = _partition_diagonals(n_t + ts.num_atoms, lane_count)
    # off[t] + t strictly increases with t: one sorted search finds every split
    rank = off + np.arange(n_t + 1, dtype=np.int64)
    tiles = np.searchsorted(rank, diag, side="right").astype(np.int64) - 1
    return np.stack([tiles, diag - tiles], axis=1)


def merge_path_slices(ts, lane_count: int) -> list[MergePathSlice]:
    c = merge_path_partition(ts, lane_count)
    return [MergePathSlice(int(c[k, 0]), int(c[k, 1]), int(c[k + 1, 0]), int(c[k + 1, 1]))
            for k in range(lane_count)]


def exclusive_prefix_sum(xs) -> np.ndarray:
    """``[x0, x1, ...] -> [0, x0, x0+x1, ...]``; negatives and int64 overflow raise."""
    counts = np.asarray(xs, dtype=np.int64).reshape(-1)
    if counts.size and int(counts.min()) < 0:
        raise ValueError("counts must be non-negative")
    out = np.empty(counts.size + 1, dtype=np.int64)
    out[0] = 0
    np.cumsum(counts, out=out[1:])
    if counts.size and bool((out[1:] < out[:-1]).any()):
        raise OverflowError("prefix sum overflows 64-bit counts")
    return out


def num_blocks(ts, tiles_per_block: int) -> int:
    return (ts.num_tiles + tiles_per_block - 1) // tiles_per_block


def group_plan(ts, group_id: int, group_count: int, tiles_per_block: int,
               block: int | None = None) -> GroupPlan:
    """Plan of one tile block owned by ``group_id`` (reference schedules.py:137-159).

    Block b covers tiles [b*tpb, min((b+1)*tpb, num_tiles)) and belongs to group
    b mod group_count; ``block`` defaults to the group's first block.
    """
    if tiles_per_block < 1:
        raise ValueError("tiles_per_block must be >= 1")
    if group_id < 0 or group_id >= group_count:
        raise ValueError("group_id must satisfy 0 <= group_id < group_count")
    b = group_id if block is None else block
    if b % group_count != group_id:
        raise ValueError(f"block {b} is not handled by group {group_id}")
    first = b * tiles_per_block
    if ts.num_tiles > 0 and first >= ts.num_tiles:
        raise ValueError(f"block {b} is past the tile range")
    count = max(0, min(tiles_per_block, ts.num_tiles - first))
    off = tile_offsets(ts)
    lengths = np.diff(off[first:first + count + 1]) if count else np.empty(0, np.int64)
    return GroupPlan(first, count, exclusive_prefix_sum(lengths))


def get_tile(plan: GroupPlan, local_atom: int) -> int:
    """Block-local tile owning ``local_atom``: prefix[t] <= a < prefix[t+1]."""
    if local_atom < 0 or local_atom >= plan.total_atoms:
        raise ValueError(f"local_atom {local_atom} outside [0, {plan.total_atoms})")
    return int(np.searchsorted(plan.prefix, local_atom, side="right")) - 1


# ---- range-based schedule objects ----------------------------------------------------

class Schedule:
    """Lane -> (tiles, atoms-of-tile) map over a tile set for ``lanes`` lanes."""

    kind: ScheduleKind

    def __init__(self, ts, lanes: int):
        if lanes < 1:
            raise ValueError("lanes must be >= 1")
        self.ts = ts
        self.lanes = int(lanes)
        self.offsets = tile_offsets(ts)

    def tiles(self, lane: int):
        raise NotImplementedError

    def atoms(self, lane: int, tile: int) -> range:
        raise NotImplementedError

    def assignment(self):
        """Yield (lane, tile, atom) for every atom, lane by lane."""
        for lane in range(self.lanes):
            for tile in self.tiles(lane):
                for atom in self.atoms(lane, tile):
                    yield lane, tile, atom


class ThreadMappedSchedule(Schedule):
    kind = ScheduleKind.THREAD_MAPPED

    def tiles(self, lane: int) -> range:
        return thread_mapped_tiles(self.ts, lane, self.lanes)

    def atoms(self, lane: int, tile: int) -> range:
        return range(int(self.offsets[tile]), int(self.offsets[tile + 1]))


class MergePathSchedule(Schedule):
    kind = ScheduleKind.MERGE_PATH

    def __init__(self, ts, lanes: int):
        super().__init__(ts, lanes)
        self.coords = merge_path_partition(ts, lanes)

    def slice(self, lane: int) -> MergePathSlice:
        c = self.coords
        return MergePathSlice(int(c[lane, 0]), int(c[lane, 1]), int(c[lane + 1, 0]),
                              int(c[lane + 1, 1]))

    def tiles(self, lane: int) -> range:
        """Tiles whose boundary the lane consumes, plus its trailing partial tile."""
        s = self.slice(lane)
        trailing = (s.tile_end < self.ts.num_tiles
                    and s.atom_end > max(s.atom_begin, int(self.offsets[s.tile_end])))
        return range(s.tile_begin, s.tile_end + (1 if trailing else 0))

    def atoms(self, lane: int, tile: int) -> range:
        s = self.slice(lane)
        lo = max(s.atom_begin, int(self.offsets[tile]))
        hi = min(s.atom_end, int(self.offsets[tile + 1]))
        return range(lo, max(lo, hi))


class GroupMappedSchedule(Schedule):
    kind = ScheduleKind.GROUP_MAPPED

    def __init__(self, ts, lanes: int, group_size: int = 32, tiles_per_block: int | None = None):
        super().__init__(ts, lanes)
        if group_size < 1:
            raise ValueError("group_size must be >= 1")
        self.group_size = int(group_size)
        self.tiles_per_block = int(tiles_per_block or group_size)
        if self.tiles_per_block < 1:
            raise ValueError("tiles_per_block must be >= 1")
        self.group_count = (self.lanes + self.group_size - 1) // self.group_size

    def _member(self, lane: int):
        gid, m = divmod(lane, self.group_size)
        members = min(self.group_size, self.lanes - gid * self.group_size)
        return gid, m, members

    def tiles(self, lane: int):
        gid, m, members = self._member(lane)
        tpb, n_t = self.tiles_per_block, self.ts.num_tiles
        for b in range(gid, num_blocks(self.ts, tpb), self.group_count):
            first, last = b * tpb, min((b + 1) * tpb, n_t)
            base = int(self.offsets[first])
            for t in range(first, last):
                if len(self._atoms(base, m, members, t)):
                    yield t

    def _atoms(self, base: int, m: int, members: int, tile: int) -> range:
        lo, hi = int(self.offsets[tile]) - base, int(self.offsets[tile + 1]) - base
        start = lo + ((m - lo) % members)
        return range(base + start, base + max(start, hi), members)

    def atoms(self, lane: int, tile: int) -> range:
        gid, m, members = self._member(lane)
        first = (tile // self.tiles_per_block) * self.tiles_per_block
        return self._atoms(int(self.offsets[first]), m, members, tile)


def make_schedule(ts, cfg) -> Schedule:
    """Schedule object for an ExecutorConfig (lanes = cfg.lanes)."""
    if cfg.schedule is ScheduleKind.THREAD_MAPPED:
        return ThreadMappedSchedule(ts, cfg.lanes)
    if cfg.schedule is ScheduleKind.MERGE_PATH:
        return MergePathSchedule(ts, cfg.lanes)
    return GroupMappedSchedule(ts, cfg.lanes, cfg.group_size, cfg.tiles_per_block)
