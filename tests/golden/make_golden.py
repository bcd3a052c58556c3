"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the dev container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the unmodified reference package (lanework 0.1.0) from
/root/reference/pkg/src and records, for seeded inputs, exactly what the
reference returns: merge-path search/partition, group plans, get_tile,
imbalance per lane, the (lane, tile) every atom is assigned to by the
reference executors, spmv results on the numba backend, and the outputs of
its synthetic generators. The .npz files it writes are committed; tests replay
them against the C oracle (CPU) and the CUDA kernels (GPU) without needing the
reference at run time.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("LANEWORK_SRC", "/root/reference/pkg/src"))
OUT = Path(__file__).resolve().parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, str(REF))

import lanework as lw  # noqa: E402  (the reference)


def tile_set_corpus(count: int, seed: int, max_tiles: int = 120, max_atoms: int = 900):
    """Empty set, a single tile, and random sets with ~25% empty tiles."""
    rng = np.random.default_rng(seed)
    out = [np.zeros(1, np.int64), np.array([0, 17], np.int64), np.array([0, 0, 0, 5], np.int64),
           np.array([0, 2, 3, 6], np.int64), np.array([0, 1000] + [1000] * 7, np.int64)]
    while len(out) < count:
        n = int(rng.integers(1, max_tiles + 1))
        counts = rng.integers(0, 2 * max_atoms // max_tiles + 1, size=n)
        counts[rng.random(n) < 0.25] = 0
        if counts.sum() > max_atoms:
            counts = counts * max_atoms // max(int(counts.sum()), 1)
        off = np.zeros(n + 1, np.int64)
        np.cumsum(counts, out=off[1:])
        out.append(off)
    return out


def pack(arrays):
    arrays = [np.asarray(a) for a in arrays]
    idx = np.zeros(len(arrays) + 1, np.int64)
    np.cumsum([a.size for a in arrays], out=idx[1:])
    flat = np.concatenate([a.reshape(-1) for a in arrays]) if arrays else np.zeros(0)
    return flat, idx


def reference_assignment(ts, cfg):
    """(lane_of_atom, tile_of_atom) exactly as the reference executors deliver atoms."""
    n = ts.num_atoms
    lane_of = np.full(n, -1, np.int64)
    tile_of = np.full(n, -1, np.int64)
    visits = np.zeros(n, np.int64)
    if cfg.schedule is lw.ScheduleKind.MERGE_PATH:
        def atom_fn(lane, tile, atom):
            lane_of[atom], tile_of[atom] = lane, tile
            visits[atom] += 1
            return 0.0

        lw.execute_merge_path(cfg, ts, atom_fn, lambda lane, tile, acc: None)
    else:
        def work_fn(lane, tile, atoms):
            for a in atoms:
                lane_of[a], tile_of[a] = lane, tile
                visits[a] += 1

        lw.execute_tile_major(cfg, ts, work_fn)
    assert (visits == 1).all()
    return lane_of, tile_of


def make_schedules():
    sets = tile_set_corpus(48, seed=1234)
    lane_counts = [1, 2, 3, 5, 7, 13, 32, 64, 100]
    search, parts, imbal, plans, tiles = [], [], [], [], []
    assign_lane, assign_tile, assign_meta = [], [], []
    gm_shapes = [(1, 1), (4, 4), (4, 7), (32, 32), (8, 3)]
    for si, off in enumerate(sets):
        ts = lw.TileSet(off)
        total = ts.num_tiles + ts.num_atoms
        search.append(np.array([lw.merge_path_search(d, ts) for d in range(total + 1)],
                               np.int64).reshape(-1, 2))
        for p in lane_counts:
            parts.append(lw.merge_path_partition(ts, p))
            for kind in lw.ScheduleKind:
                shapes = gm_shapes if kind is lw.ScheduleKind.GROUP_MAPPED else [(32, 32)]
                for gs, tpb in shapes:
                    cfg = lw.ExecutorConfig(schedule=kind, lanes=p, group_size=gs,
                                            tiles_per_block=tpb)
                    imbal.append(lw.imbalance(ts, cfg).per_lane_atoms)
                    if p in (1, 3, 7, 32) and si < 24:
                        lo, to = reference_assignment(ts, cfg)
                        assign_lane.append(lo)
                        assign_tile.append(to)
                        assign_meta.append([si, p, list(lw.ScheduleKind).index(kind), gs, tpb])
        for tpb in (1, 3, 32):
            nb = lw.schedules.num_blocks(ts, tpb)
            for b in range(nb):
                plan = lw.group_plan(ts, b, nb, tpb, block=b)
                plans.append(plan.prefix)
                tiles.append(np.array([lw.get_tile(plan, a) for a in range(plan.total_atoms)],
                                      np.int64))
    np.savez_compressed(
        OUT / "schedules.npz",
        sets=pack(sets)[0], sets_idx=pack(sets)[1], lane_counts=np.array(lane_counts),
        search=pack(search)[0], search_idx=pack(search)[1],
        parts=pack(parts)[0], parts_idx=pack(parts)[1],
        imbal=pack(imbal)[0], imbal_idx=pack(imbal)[1],
        gm_shapes=np.array(gm_shapes),
        plans=pack(plans)[0], plans_idx=pack(plans)[1],
        tiles=pack(tiles)[0], tiles_idx=pack(tiles)[1],
        assign_lane=pack(assign_lane)[0], assign_tile=pack(assign_tile)[0],
        assign_idx=pack(assign_lane)[1], assign_meta=np.array(assign_meta, np.int64),
    )


def make_spmv():
    rng = np.random.default_rng(2024)
    mats, xs, ys, meta = [], [], [], []
    cfgs = []
    for lanes in (9, 16, 64):
        cfgs.append(("thread-mapped", lanes, 32, 32))
        cfgs.append(("merge-path", lanes, 32, 32))
        for gs in (4, 32, 256):
            cfgs.append(("group-mapped", lanes, gs, gs))
    for i in range(24):
        rows = int(rng.integers(1, 120))
        cols = int(rng.integers(1, 120))
        nnz = int(rng.integers(0, min(rows * cols, 900) + 1))
        m = lw.generate_random_csr(rows, cols, nnz, seed=int(rng.integers(1 << 30)))
        integer = i % 2 == 0
        if integer:
            m.values = rng.integers(-4, 5, size=m.nnz).astype(np.float64)
            x = rng.integers(-3, 4, size=cols).astype(np.float64)
        else:
            x = rng.random(cols)
        for ci, (kind, lanes, gs, tpb) in enumerate(cfgs):
            cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind(kind), lanes=lanes, worker_threads=2,
                                    group_size=gs, tiles_per_block=tpb)
            ys.append(lw.spmv(m, x, cfg))
            meta.append([i, ci, int(integer)])
        mats.append(m)
        xs.append(x)
    np.savez_compressed(
        OUT / "spmv.npz",
        rows=np.array([m.rows for m in mats]), cols=np.array([m.cols for m in mats]),
        off=pack([m.row_offsets for m in mats])[0], off_idx=pack([m.row_offsets for m in mats])[1],
        col=pack([m.col_indices for m in mats])[0], col_idx=pack([m.col_indices for m in mats])[1],
        val=pack([m.values for m in mats])[0],
        x=pack(xs)[0], x_idx=pack(xs)[1],
        y=pack(ys)[0], y_idx=pack(ys)[1], meta=np.array(meta),
        cfg_kind=np.array([c[0] for c in cfgs]), cfg_lanes=np.array([c[1] for c in cfgs]),
        cfg_gs=np.array([c[2] for c in cfgs]), cfg_tpb=np.array([c[3] for c in cfgs]),
    )


def make_spmm():
    """spmm outputs (numba backend) for seeded matrices x dense B (kernels.py:129-175)."""
    rng = np.random.default_rng(2025)
    mats, bs, cs, meta = [], [], [], []
    cfgs = []
    for lanes in (5, 16, 64):
        cfgs.append(("thread-mapped", lanes, 32, 32))
        cfgs.append(("merge-path", lanes, 32, 32))
        for gs in (4, 32):
            cfgs.append(("group-mapped", lanes, gs, gs))
    for i in range(16):
        rows = int(rng.integers(1, 90))
        cols = int(rng.integers(1, 90))
        nnz = int(rng.integers(0, min(rows * cols, 700) + 1))
        m = lw.generate_random_csr(rows, cols, nnz, seed=int(rng.integers(1 << 30)))
        n = [1, 2, 3, 4, 8, 5, 16, 33][i % 8]
        integer = i % 2 == 0
        if integer:
            m.values = rng.integers(-4, 5, size=m.nnz).astype(np.float64)
            B = rng.integers(-3, 4, size=(cols, n)).astype(np.float64)
        else:
            B = rng.random((cols, n))
        for ci, (kind, lanes, gs, tpb) in enumerate(cfgs):
            cfg = lw.ExecutorConfig(schedule=lw.ScheduleKind(kind), lanes=lanes, worker_threads=2,
                                    group_size=gs, tiles_per_block=tpb)
            cs.append(lw.spmm(m, B, cfg))
            meta.append([i, ci, int(integer)])
        mats.append(m)
        bs.append(B)
    np.savez_compressed(
        OUT / "spmm.npz",
        rows=np.array([m.rows for m in mats]), cols=np.array([m.cols for m in mats]),
        n=np.array([b.shape[1] for b in bs]),
        off=pack([m.row_offsets for m in mats])[0], off_idx=pack([m.row_offsets for m in mats])[1],
        col=pack([m.col_indices for m in mats])[0], col_idx=pack([m.col_indices for m in mats])[1],
        val=pack([m.values for m in mats])[0],
        B=pack(bs)[0], B_idx=pack(bs)[1],
        C=pack(cs)[0], C_idx=pack(cs)[1], meta=np.array(meta),
        cfg_kind=np.array([c[0] for c in cfgs]), cfg_lanes=np.array([c[1] for c in cfgs]),
        cfg_gs=np.array([c[2] for c in cfgs]), cfg_tpb=np.array([c[3] for c in cfgs]),
    )


def _mm_text(rng, k):
    """A Matrix Market text with the variety real files have: every field and
    symmetry, comments and blank lines, ragged whitespace, CRLF, duplicates,
    unsorted entries, exponents."""
    field = ["real", "integer", "pattern"][k % 3]
    sym = "symmetric" if k % 4 == 1 else "general"
    rows = int(rng.integers(1, 40))
    cols = rows if sym == "symmetric" else int(rng.integers(1, 40))
    n = int(rng.integers(0, 3 * max(rows, cols) + 1))
    lines = [f"%%MatrixMarket {'Matrix' if k % 5 == 0 else 'matrix'} coordinate {field} {sym}"]
    if k % 3 == 0:
        lines += ["% generated", ""]
    lines.append(f"{rows} {cols} {n}")
    for e in range(n):
        i = int(rng.integers(1, rows + 1))
        j = int(rng.integers(1, cols + 1))
        if sym == "symmetric" and j > i:
            i, j = j, i
        sep = "\t" if (e + k) % 7 == 0 else " " * int(rng.integers(1, 3))
        if field == "pattern":
            lines.append(f"{i}{sep}{j}")
        elif field == "integer":
            lines.append(f"{i}{sep}{j}{sep}{int(rng.integers(-9, 10))}")
        else:
            v = float(rng.normal()) * 10.0 ** int(rng.integers(-5, 6))
            lines.append(f"{i}{sep}{j}{sep}{v!r}" if e % 3 else f"{i} {j} {v:.6e}")
        if e % 11 == 5:
            lines.append("% interleaved comment")
    nl = "\r\n" if k % 6 == 2 else "\n"
    return nl.join(lines) + nl


MM_ERROR_TEXTS = [
    "",
    "%%NotMatrixMarket matrix coordinate real general\n1 1 0\n",
    "%%MatrixMarket matrix coordinate real\n1 1 0\n",
    "%%MatrixMarket tensor coordinate real general\n1 1 0\n",
    "%%MatrixMarket matrix array real general\n1 1\n",
    "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "%%MatrixMarket matrix coordinate real general\n2 -2 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 x 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 2.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\nx y z\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 0 1.0\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\nx y z\n",
    "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n1 1 1\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n1 2 abc\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 5 1.0\n1 x 1\n",
    "%%MatrixMarket matrix coordinate integer general\n3 3 1\n1.5 1 2\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 0x10\n",
]


def make_mmio():
    """parse_matrix_market + coo_to_csr outputs, and the error message of every
    malformed text (mmio.py:24-107, sparse.py:130-150)."""
    from lanework.mmio import MatrixMarketError

    rng = np.random.default_rng(77)
    texts, coo_r, coo_c, coo_v, shapes, offs, cols_, vals_ = [], [], [], [], [], [], [], []
    for k in range(36):
        t = _mm_text(rng, k)
        coo = lw.parse_matrix_market(t)
        csr = lw.coo_to_csr(coo)
        texts.append(t)
        coo_r.append(coo.row)
        coo_c.append(coo.col)
        coo_v.append(coo.data)
        shapes.append([coo.rows, coo.cols])
        offs.append(csr.row_offsets)
        cols_.append(csr.col_indices)
        vals_.append(csr.values)
    msgs = []
    for t in MM_ERROR_TEXTS:
        try:
            lw.parse_matrix_market(t)
            msgs.append("")
        except MatrixMarketError as exc:
            msgs.append(str(exc))
    np.savez_compressed(
        OUT / "mmio.npz", texts=np.array(texts), shapes=np.array(shapes),
        coo_r=pack(coo_r)[0], coo_c=pack(coo_c)[0], coo_v=pack(coo_v)[0], coo_idx=pack(coo_r)[1],
        off=pack(offs)[0], off_idx=pack(offs)[1], col=pack(cols_)[0], val=pack(vals_)[0],
        col_idx=pack(cols_)[1], err_texts=np.array(MM_ERROR_TEXTS), err_msgs=np.array(msgs))


def make_traversal():
    """sssp / bfs (numba) and the serial references dijkstra / serial_bfs
    (kernels.py:320-357, reference.py) on graphs with unreachable parts,
    self-loops, integer and real non-negative weights."""
    from lanework import reference as ref

    rng = np.random.default_rng(99)
    offs, cols, ws, srcs, dists, dijk, depths, sbfs = [], [], [], [], [], [], [], []
    for k in range(14):
        n = int(rng.integers(2, 300))
        if k % 3 == 0:
            m = lw.generate_power_law_csr(n, 4.0, 1.3, seed=int(rng.integers(1 << 30)))
        else:
            m = lw.generate_random_csr(n, n, int(rng.integers(0, min(n * n, 6 * n) + 1)),
                                       seed=int(rng.integers(1 << 30)))
        if k % 2 == 0:
            m.values = rng.integers(0, 10, size=m.nnz).astype(np.float64)
        else:
            m.values = np.abs(m.values)
        g = lw.Graph(m)
        src = int(rng.integers(0, n))
        offs.append(m.row_offsets)
        cols.append(m.col_indices)
        ws.append(m.values)
        srcs.append(src)
        dists.append(lw.sssp(g, src))
        dijk.append(ref.dijkstra(g, src))
        depths.append(lw.bfs(g, src))
        sbfs.append(ref.serial_bfs(g, src))
    np.savez_compressed(
        OUT / "traversal.npz", off=pack(offs)[0], off_idx=pack(offs)[1], col=pack(cols)[0],
        w=pack(ws)[0], col_idx=pack(cols)[1], src=np.array(srcs),
        dist=pack(dists)[0], dijkstra=pack(dijk)[0], depth=pack(depths)[0],
        serial_bfs=pack(sbfs)[0], v_idx=pack(dists)[1])


def make_generators():
    out = {}
    cases = [("random", (40, 30, 200, 1)), ("random", (300, 200, 5000, 7)),
             ("random", (5000, 5000, 10000, 11)), ("random", (10, 10, 100, 3)),
             ("power", (500, 8.0, 1.1, 3)), ("power", (2000, 16.0, 1.5, 4)),
             ("power", (1000, 4.0, 3.0, 5))]
    for k, (kind, args) in enumerate(cases):
        m = lw.generate_random_csr(*args) if kind == "random" else lw.generate_power_law_csr(*args)
        out[f"c{k}_kind"] = np.array(kind)
        out[f"c{k}_args"] = np.array(args, dtype=np.float64)
        out[f"c{k}_off"] = m.row_offsets
        out[f"c{k}_col"] = m.col_indices
        out[f"c{k}_val"] = m.values
    out["count"] = np.array(len(cases))
    np.savez_compressed(OUT / "generators.npz", **out)


if __name__ == "__main__":
    print("reference:", lw.__file__, "backend:", lw.backend_name())
    names = ("schedules", "spmv", "spmm", "mmio", "traversal", "generators")
    which = set(sys.argv[1:]) or set(names)
    for name in names:
        if name in which:
            globals()[f"make_{name}"]()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
