"""SSSP and BFS on the cuda backend (reference kernels.py:230-381).

Same names and behaviour as the reference: ``sssp(g, source, cfg)`` returns
float64 distances (+inf unreached), ``bfs(g, source, cfg)`` int64 hop counts
(``UNREACHED`` = -1), ``sssp_init`` / ``sssp_pass`` expose one relaxation pass
with its frontier masks (the caller owns the convergence loop), and a pass
returns how many vertices entered the next frontier. ``g`` is a
:class:`~paper_2301_04792_b200.sparse.Graph` (host, weights uploaded as fp64 like
the reference computes) or a square :class:`DeviceCsr` (fp32/fp64 weights,
results stay on the device as torch tensors).

Every pass runs on the device through the C ABI (lw_frontier_compact,
lw_sssp_pass / lw_bfs_pass, lw_sssp / lw_bfs): ordered frontier compaction,
the frontier tile set (tiles = active vertices, atoms = out-edges) and the
schedule's relaxation kernel. The schedule decides which lane relaxes which
edge; the distances do not depend on it (see csrc/frontier.cu).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _backend, _lib
from .device import DeviceCsr, Workspace, cached_device_csr, current_stream
from .executor import ExecutorConfig
from .kernels import schedule_code
from .sparse import Graph

__all__ = ["UNREACHED", "SsspState", "sssp_init", "sssp_pass", "sssp", "bfs", "bfs_pass",
           "device_graph"]

UNREACHED = -1

_WS = Workspace()


def device_graph(g, dtype="float64") -> DeviceCsr:
    """A Graph (host) uploaded as a square DeviceCsr, or a DeviceCsr checked the
    way reference Graph checks a host matrix (sparse.py:114-118): square, and no
    negative edge weight (the SSSP kernels' atomicMin on the fp64 bit pattern is
    only an order-preserving min for non-negative values). The weight check is
    one device reduction per values tensor, remembered while that tensor is the
    same object at the same version."""
    if isinstance(g, DeviceCsr):
        if g.rows != g.cols:
            raise ValueError("adjacency matrix must be square")
        v = g.values
        seen = g.__dict__.get("_nonneg_checked")
        if seen is None or seen[0] is not v or seen[1] != v._version:
            if g.nnz and bool((v < 0).any().item()):
                raise ValueError("edge weights must be non-negative")
            g.__dict__["_nonneg_checked"] = (v, v._version)
        return g
    if not isinstance(g, Graph):
        g = Graph(g)
    return cached_device_csr(g.csr, dtype=dtype)


def _ws(G: DeviceCsr):
    need = _lib.load().lw_frontier_workspace(G.rows)
    return _WS.get(need, G.device, current_stream(G.device)), need


def _cfg_args(cfg: ExecutorConfig):
    return (schedule_code(cfg.schedule), 0 if cfg.lanes_auto else int(cfg.lanes),
            cfg.group_size, cfg.tiles_per_block)


def _check_source(n: int, source: int):
    if not 0 <= source < n:
        raise ValueError(f"source {source} outside [0, {n})")


@dataclass
class SsspState:
    """Distances plus the current and next frontier masks (reference kernels.py:230-236)."""

    dist: object
    in_frontier: object
    out_frontier: object


def sssp_init(num_vertices: int, source: int) -> SsspState:
    _check_source(num_vertices, source)
    dist = np.full(num_vertices, np.inf)
    dist[source] = 0.0
    in_frontier = np.zeros(num_vertices, dtype=bool)
    in_frontier[source] = True
    return SsspState(dist, in_frontier, np.zeros(num_vertices, dtype=bool))


def _compact(G: DeviceCsr, mask, ws, need, stream):
    import torch

    active = torch.empty(max(G.rows, 1), dtype=torch.int32, device=G.device)
    count = torch.zeros(1, dtype=torch.int64, device=G.device)
    rc = _lib.load().lw_frontier_compact(mask.data_ptr(), G.rows, active.data_ptr(),
                                         count.data_ptr(), ws.data_ptr(), need, stream)
    _lib.check(rc, "lw_frontier_compact")
    return active, int(count.item())


def sssp_pass(g, state: SsspState, cfg: ExecutorConfig | None = None) -> int:
    """Relax every out-edge of the current frontier once (reference kernels.py:245-268).

    A vertex joins ``out_frontier`` only when its distance strictly improved.
    Host states (NumPy arrays) are updated in place; device states (torch
    tensors: fp64 dist, uint8/bool masks) stay on the device."""
    cfg = cfg or ExecutorConfig()
    _backend.require_cuda()
    import torch

    G = device_graph(g)
    host = isinstance(state.dist, np.ndarray)
    dev = G.device
    dist = torch.as_tensor(state.dist).to(dev, torch.float64).contiguous() if host else state.dist
    inm = torch.as_tensor(np.asarray(state.in_frontier)).to(dev, torch.uint8) if host \
        else state.in_frontier.to(torch.uint8)
    out = torch.empty(G.rows, dtype=torch.uint8, device=dev)
    ws, need = _ws(G)
    stream = current_stream(dev)
    active, n_active = _compact(G, inm, ws, need, stream)
    code, lanes, gs, tpb = _cfg_args(cfg)
    rc = _lib.load().lw_sssp_pass(G.c_struct(), active.data_ptr(), n_active, dist.data_ptr(),
                                  out.data_ptr(), code, lanes, gs, tpb, ws.data_ptr(), need, stream)
    _lib.check(rc, "lw_sssp_pass")
    count = int(out.sum().item())
    if host:
        state.dist[:] = dist.cpu().numpy()
        state.out_frontier = out.bool().cpu().numpy()
    else:
        state.dist = dist
        state.out_frontier = out.bool()
    return count


def bfs_pass(g, depth, frontier, next_depth: int, cfg: ExecutorConfig | None = None):
    """One level of BFS on device tensors: claims unvisited neighbours of the
    frontier with ``next_depth``; returns the next frontier (bool tensor)."""
    cfg = cfg or ExecutorConfig()
    _backend.require_cuda()
    import torch

    G = device_graph(g)
    out = torch.empty(G.rows, dtype=torch.uint8, device=G.device)
    ws, need = _ws(G)
    stream = current_stream(G.device)
    active, n_active = _compact(G, frontier.to(torch.uint8), ws, need, stream)
    code, lanes, gs, tpb = _cfg_args(cfg)
    rc = _lib.load().lw_bfs_pass(G.c_struct(), active.data_ptr(), n_active, depth.data_ptr(),
                                 next_depth, out.data_ptr(), code, lanes, gs, tpb, ws.data_ptr(),
                                 need, stream)
    _lib.check(rc, "lw_bfs_pass")
    return out.bool()


def _traverse(g, source: int, cfg: ExecutorConfig | None, bfs_mode: bool, return_passes: bool):
    cfg = cfg or ExecutorConfig()
    _backend.require_cuda()
    import torch

    host = not isinstance(g, DeviceCsr)
    G = device_graph(g)
    _check_source(G.rows, source)
    out = torch.empty(G.rows, dtype=torch.int64 if bfs_mode else torch.float64, device=G.device)
    ws, need = _ws(G)
    passes = ctypes.c_int64(0)
    code, lanes, gs, tpb = _cfg_args(cfg)
    fn = _lib.load().lw_bfs if bfs_mode else _lib.load().lw_sssp
    rc = fn(G.c_struct(), source, out.data_ptr(), code, lanes, gs, tpb, ws.data_ptr(), need,
            ctypes.byref(passes), current_stream(G.device))
    _lib.check(rc, "lw_bfs" if bfs_mode else "lw_sssp")
    res = out.cpu().numpy() if host else out
    return (res, passes.value) if return_passes else res


def sssp(g, source: int, cfg: ExecutorConfig | None = None, *, return_passes: bool = False):
    """Single-source shortest distances by frontier relaxation; unreached vertices
    keep +inf (reference kernels.py:320-327). Weights must be non-negative."""
    return _traverse(g, source, cfg, False, return_passes)


def bfs(g, source: int, cfg: ExecutorConfig | None = None, *, return_passes: bool = False):
    """Hop counts from ``source``; unreached vertices get UNREACHED (kernels.py:330-357)."""
    return _traverse(g, source, cfg, True, return_passes)
