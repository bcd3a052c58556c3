/*
 * lw_oracle.c — TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of the reference's SpMV path (lanework 0.1.0,
 * /root/reference/pkg/src/lanework) in plain C + OpenMP, used by tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm. Nothing
 * under paper_2301_04792_b200/ links or calls this file.
 *
 * Semantics follow the reference exactly (fp64 arithmetic on int64 offsets,
 * int64 column indices and float64 values — the reference's only precision,
 * sparse.py:55-58, kernels.py:60-63), including its lane model: P virtual lanes
 * sharded round-robin over T worker threads (executor.py:107-129).
 * Pinned against the reference's own outputs by tests/golden (make_golden.py
 * imports the reference and records partitions, plans, per-lane counts,
 * assignment maps and SpMV results; tests/test_oracle_golden.py replays them).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/lw_hash.h"

#define EXPORT __attribute__((visibility("default")))

static int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

EXPORT int lwo_version(void) { return 1; }

/* schedules.py:63-85 — greatest t in [max(0,d-nnz), min(d,rows)] with off[t] <= d-t */
EXPORT int64_t lwo_merge_path_search(const int64_t* off, int64_t rows, int64_t nnz, int64_t d) {
    int64_t lo = imax(0, d - nnz), hi = imin(d, rows);
    while (lo < hi) {
        int64_t mid = (lo + hi + 1) / 2;
        if (off[mid] <= d - mid) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

/* schedules.py:88-110 — coords[2k] = tile_k, coords[2k+1] = atom_k */
EXPORT void lwo_merge_path_partition(const int64_t* off, int64_t rows, int64_t nnz, int64_t lanes,
                                     int64_t* coords, int threads) {
    const int64_t total = rows + nnz;
    const int64_t items = total ? (total + lanes - 1) / lanes : 0;
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t k = 0; k <= lanes; ++k) {
        int64_t d = imin(k * items, total);
        int64_t t = lwo_merge_path_search(off, rows, nnz, d);
        coords[2 * k] = t;
        coords[2 * k + 1] = d - t;
    }
}

/* _fast.py:20-28 + kernels.py:74-79 — thread j runs lanes j, j+T, ...; lane l
 * owns tiles l, l+P, ... and assigns y[t] from a sequential fp64 sum. */
EXPORT void lwo_spmv_thread_mapped(const int64_t* off, const int64_t* col, const double* val,
                                   const double* x, double* y, int64_t rows, int64_t lanes,
                                   int threads) {
#pragma omp parallel num_threads(threads)
    {
        const int j = omp_get_thread_num(), T = omp_get_num_threads();
        for (int64_t lane = j; lane < lanes; lane += T)
            for (int64_t t = lane; t < rows; t += lanes) {
                double acc = 0.0;
                for (int64_t a = off[t]; a < off[t + 1]; ++a) acc += val[a] * x[col[a]];
                y[t] = acc;
            }
    }
}

/* _fast.py:31-52 + kernels.py:80-91 — host partition, per-lane slices with
 * carries, then the serial fix-up in lane order. coords may be NULL (computed
 * here) or a caller buffer of (lanes+1)*2 int64 to reuse. */
EXPORT int lwo_spmv_merge_path(const int64_t* off, const int64_t* col, const double* val,
                               const double* x, double* y, int64_t rows, int64_t nnz,
                               int64_t lanes, int threads, int64_t* coords_buf) {
    int64_t* coords = coords_buf ? coords_buf : (int64_t*)malloc(sizeof(int64_t) * 2 * (lanes + 1));
    int64_t* carry_tile = (int64_t*)malloc(sizeof(int64_t) * lanes);
    double* carry_val = (double*)malloc(sizeof(double) * lanes);
    if (!coords || !carry_tile || !carry_val) return -1;
    lwo_merge_path_partition(off, rows, nnz, lanes, coords, threads);
#pragma omp parallel num_threads(threads)
    {
        const int j = omp_get_thread_num(), T = omp_get_num_threads();
        for (int64_t lane = j; lane < lanes; lane += T) {
            int64_t atom = coords[2 * lane + 1];
            const int64_t tile_end = coords[2 * lane + 2], atom_end = coords[2 * lane + 3];
            double acc = 0.0;
            for (int64_t t = coords[2 * lane]; t < tile_end; ++t) {
                for (; atom < off[t + 1]; ++atom) acc += val[atom] * x[col[atom]];
                y[t] = acc;
                acc = 0.0;
            }
            carry_tile[lane] = -1;
            carry_val[lane] = 0.0;
            if (atom < atom_end) {
                for (; atom < atom_end; ++atom) acc += val[atom] * x[col[atom]];
                carry_tile[lane] = tile_end;
                carry_val[lane] = acc;
            }
        }
    }
    for (int64_t lane = 0; lane < lanes; ++lane)
        if (carry_tile[lane] >= 0) y[carry_tile[lane]] += carry_val[lane];
    if (!coords_buf) free(coords);
    free(carry_tile);
    free(carry_val);
    return 0;
}

/* _fast.py:55-77 + kernels.py:92-98 — group g (members = min(gs, P-g*gs)) owns
 * blocks g, g+G, ...; member m takes local atoms m, m+members, ...; y pre-zeroed
 * and accumulated with +=. Groups are sharded over threads like group_shards. */
EXPORT void lwo_spmv_group_mapped(const int64_t* off, const int64_t* col, const double* val,
                                  const double* x, double* y, int64_t rows, int64_t lanes,
                                  int64_t gs, int64_t tpb, int threads) {
    const int64_t groups = (lanes + gs - 1) / gs;
    const int64_t blocks = (rows + tpb - 1) / tpb;
    memset(y, 0, sizeof(double) * rows);
#pragma omp parallel num_threads(threads)
    {
        const int j = omp_get_thread_num(), T = omp_get_num_threads();
        for (int64_t g = j; g < groups; g += T) {
            const int64_t members = imin(gs, lanes - g * gs);
            if (members <= 0) continue;
            for (int64_t b = g; b < blocks; b += groups) {
                const int64_t tb = b * tpb, tc = imin(tpb, rows - tb);
                const int64_t base = off[tb], total = off[tb + tc] - base;
                for (int64_t m = 0; m < members; ++m) {
                    int64_t t = tb;
                    for (int64_t k = m; k < total; k += members) {
                        const int64_t a = base + k;
                        while (off[t + 1] <= a) ++t;
                        y[t] += val[a] * x[col[a]];
                    }
                }
            }
        }
    }
}

/* ---- SpMM: C = A B, B row-major [cols x n], C row-major [rows x n] ----------
 * The column loop wraps the SpMV body (Listing 4; kernels.py:129-175). */

/* _fast.py:80-90 — lane l owns tiles l, l+P, ...; per column a sequential fp64 sum */
EXPORT void lwo_spmm_thread_mapped(const int64_t* off, const int64_t* col, const double* val,
                                   const double* B, double* C, int64_t rows, int64_t n,
                                   int64_t lanes, int threads) {
#pragma omp parallel num_threads(threads)
    {
        const int j = omp_get_thread_num(), T = omp_get_num_threads();
        for (int64_t lane = j; lane < lanes; lane += T)
            for (int64_t t = lane; t < rows; t += lanes)
                for (int64_t c = 0; c < n; ++c) {
                    double acc = 0.0;
                    for (int64_t a = off[t]; a < off[t + 1]; ++a) acc += val[a] * B[col[a] * n + c];
                    C[t * n + c] = acc;
                }
    }
}

/* _fast.py:93-118 + kernels.py:153-163 — per-lane slices; the trailing partial
 * row becomes a carry row of n values; carries added in lane order. */
EXPORT int lwo_spmm_merge_path(const int64_t* off, const int64_t* col, const double* val,
                               const double* B, double* C, int64_t rows, int64_t nnz, int64_t n,
                               int64_t lanes, int threads) {
    int64_t* coords = (int64_t*)malloc(sizeof(int64_t) * 2 * (lanes + 1));
    int64_t* carry_tile = (int64_t*)malloc(sizeof(int64_t) * lanes);
    double* carry_val = (double*)calloc((size_t)(lanes * (n > 0 ? n : 1)), sizeof(double));
    if (!coords || !carry_tile || !carry_val) { free(coords); free(carry_tile); free(carry_val); return -1; }
    lwo_merge_path_partition(off, rows, nnz, lanes, coords, threads);
#pragma omp parallel num_threads(threads)
    {
        const int j = omp_get_thread_num(), T = omp_get_num_threads();
        for (int64_t lane = j; lane < lanes; lane += T) {
            const int64_t atom_begin = coords[2 * lane + 1];
            const int64_t tile_end = coords[2 * lane + 2], atom_end = coords[2 * lane + 3];
            int64_t atom = atom_begin;
            for (int64_t t = coords[2 * lane]; t < tile_end; ++t) {
                const int64_t row_end = off[t + 1];
                for (int64_t c = 0; c < n; ++c) {
                    double acc = 0.0;
                    for (int64_t a = atom; a < row_end; ++a) acc += val[a] * B[col[a] * n + c];
                    C[t * n + c] = acc;
                }
                atom = row_end;
            }
            carry_tile[lane] = -1;
            if (atom < atom_end) {
                carry_tile[lane] = tile_end;
                for (int64_t c = 0; c < n; ++c) {
                    double acc = 0.0;
                    for (int64_t a = atom; a < atom_end; ++a) acc += val[a] * B[col[a] * n + c];
                    carry_val[lane * n + c] = acc;
                }
            }
        }
    }
    for (int64_t lane = 0; lane < lanes; ++lane)
        if (carry_tile[lane] >= 0)
            for (int64_t c = 0; c < n; ++c) C[carry_tile[lane] * n + c] += carry_val[lane * n + c];
    free(coords);
    free(carry_tile);
    free(carry_val);
    return 0;
}

/* _fast.py:121-144 — group-mapped member loop, C pre-zeroed and accumulated */
EXPORT void lwo_spmm_group_mapped(const int64_t* off, const int64_t* col, const double* val,
                                  const double* B, double* C, int64_t rows, int64_t n,
                                  int64_t lanes, int64_t gs, int64_t tpb, int threads) {
    const int64_t groups = (lanes + gs - 1) / gs;
    const int64_t blocks = (rows + tpb - 1) / tpb;
    memset(C, 0, sizeof(double) * (size_t)(rows * n));
#pragma omp parallel num_threads(threads)
    {
        const int j = omp_get_thread_num(), T = omp_get_num_threads();
        for (int64_t g = j; g < groups; g += T) {
            const int64_t members = imin(gs, lanes - g * gs);
            if (members <= 0) continue;
            for (int64_t b = g; b < blocks; b += groups) {
                const int64_t tb = b * tpb, tc = imin(tpb, rows - tb);
                const int64_t base = off[tb], total = off[tb + tc] - base;
                for (int64_t m = 0; m < members; ++m) {
                    int64_t t = tb;
                    for (int64_t k = m; k < total; k += members) {
                        const int64_t a = base + k;
                        while (off[t + 1] <= a) ++t;
                        const double v = val[a];
                        const double* src = B + col[a] * n;
                        for (int64_t c = 0; c < n; ++c) C[t * n + c] += v * src[c];
                    }
                }
            }
        }
    }
}

/* ---- SSSP / BFS (kernels.py:320-357 driving _fast.py:147-170) -------------------
 * Frontier passes: active = flatnonzero(in_frontier) in vertex order, every
 * out-edge relaxed serially, until the frontier is empty. Return the pass count. */
EXPORT int64_t lwo_sssp(const int64_t* off, const int64_t* col, const double* w, int64_t n,
                        int64_t src, double* dist) {
    unsigned char* in = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
    unsigned char* out = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
    if (!in || !out) { free(in); free(out); return -1; }
    for (int64_t i = 0; i < n; ++i) dist[i] = __builtin_inf();
    dist[src] = 0.0;
    in[src] = 1;
    int64_t passes = 0;
    for (;;) {
        int any = 0;
        memset(out, 0, (size_t)n);
        for (int64_t u = 0; u < n; ++u) {
            if (!in[u]) continue;
            any = 1;
            const double du = dist[u];
            for (int64_t e = off[u]; e < off[u + 1]; ++e) {
                const int64_t v = col[e];
                const double nd = du + w[e];
                if (nd < dist[v]) { dist[v] = nd; out[v] = 1; }
            }
        }
        if (!any) break;
        ++passes;
        unsigned char* t = in; in = out; out = t;
    }
    free(in);
    free(out);
    return passes;
}

EXPORT int64_t lwo_bfs(const int64_t* off, const int64_t* col, int64_t n, int64_t src,
                       int64_t* depth) {
    unsigned char* in = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
    unsigned char* out = (unsigned char*)calloc((size_t)(n > 0 ? n : 1), 1);
    if (!in || !out) { free(in); free(out); return -1; }
    for (int64_t i = 0; i < n; ++i) depth[i] = -1;
    depth[src] = 0;
    in[src] = 1;
    int64_t level = 0;
    for (;;) {
        int any = 0;
        memset(out, 0, (size_t)n);
        for (int64_t u = 0; u < n; ++u) {
            if (!in[u]) continue;
            any = 1;
            for (int64_t e = off[u]; e < off[u + 1]; ++e) {
                const int64_t v = col[e];
                if (depth[v] < 0) { depth[v] = level + 1; out[v] = 1; }
            }
        }
        if (!any) break;
        ++level;
        unsigned char* t = in; in = out; out = t;
    }
    free(in);
    free(out);
    return level;
}

/* ---- assignment maps (executor.py:132-209, 224-251) ------------------------
 * For every atom: the lane that processes it and the tile it is attributed to;
 * per lane: how many atoms it processes. Arrays may be NULL. lane_atoms is
 * zeroed here. */
EXPORT void lwo_assign_thread_mapped(const int64_t* off, int64_t rows, int64_t lanes,
                                     int64_t* lane_atoms, int32_t* atom_lane, int32_t* atom_tile) {
    if (lane_atoms) memset(lane_atoms, 0, sizeof(int64_t) * lanes);
    for (int64_t t = 0; t < rows; ++t) {
        const int64_t lane = t % lanes;
        if (lane_atoms) lane_atoms[lane] += off[t + 1] - off[t];
        for (int64_t a = off[t]; a < off[t + 1]; ++a) {
            if (atom_lane) atom_lane[a] = (int32_t)lane;
            if (atom_tile) atom_tile[a] = (int32_t)t;
        }
    }
}

EXPORT void lwo_assign_merge_path(const int64_t* off, int64_t rows, int64_t nnz, int64_t lanes,
                                  int64_t* lane_atoms, int32_t* atom_lane, int32_t* atom_tile) {
    int64_t* coords = (int64_t*)malloc(sizeof(int64_t) * 2 * (lanes + 1));
    lwo_merge_path_partition(off, rows, nnz, lanes, coords, 1);
    for (int64_t lane = 0; lane < lanes; ++lane) {
        int64_t atom = coords[2 * lane + 1];
        const int64_t tile_end = coords[2 * lane + 2], atom_end = coords[2 * lane + 3];
        if (lane_atoms) lane_atoms[lane] = atom_end - atom;
        int64_t t = coords[2 * lane];
        for (; atom < atom_end; ++atom) {
            while (t < tile_end && off[t + 1] <= atom) ++t;
            if (atom_lane) atom_lane[atom] = (int32_t)lane;
            if (atom_tile) atom_tile[atom] = (int32_t)t;
        }
    }
    free(coords);
}

EXPORT void lwo_assign_group_mapped(const int64_t* off, int64_t rows, int64_t lanes, int64_t gs,
                                    int64_t tpb, int64_t* lane_atoms, int32_t* atom_lane,
                                    int32_t* atom_tile) {
    const int64_t groups = (lanes + gs - 1) / gs;
    const int64_t blocks = (rows + tpb - 1) / tpb;
    if (lane_atoms) memset(lane_atoms, 0, sizeof(int64_t) * lanes);
    for (int64_t b = 0; b < blocks; ++b) {
        const int64_t g = b % groups;
        const int64_t members = imin(gs, lanes - g * gs);
        if (members <= 0) continue;
        const int64_t tb = b * tpb, tc = imin(tpb, rows - tb);
        const int64_t base = off[tb], total = off[tb + tc] - base;
        int64_t t = tb;
        for (int64_t k = 0; k < total; ++k) {
            const int64_t a = base + k, lane = g * gs + k % members;
            while (off[t + 1] <= a) ++t;
            if (lane_atoms) lane_atoms[lane] += 1;
            if (atom_lane) atom_lane[a] = (int32_t)lane;
            if (atom_tile) atom_tile[a] = (int32_t)t;
        }
    }
}

/* ---- synthetic inputs: the same counter-based functions as the device ------ */
EXPORT void lwo_rmat_keys(int scale, int64_t edge_begin, int64_t n_edges, uint32_t ta,
                          uint32_t tab, uint32_t tabc, uint64_t seed, int64_t* keys, int threads) {
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n_edges; ++i)
        keys[i] = (int64_t)lw_rmat_key(seed, (uint64_t)(edge_begin + i), scale, ta, tab, tabc);
}

EXPORT void lwo_uniform_keys(int64_t space, int64_t begin, int64_t n, uint64_t seed, int64_t* keys,
                             int threads) {
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n; ++i) keys[i] = (int64_t)lw_uniform_key(seed, (uint64_t)(begin + i), (uint64_t)space);
}

EXPORT void lwo_hash_values(const int64_t* keys, int64_t n, uint64_t seed, double* out,
                            int threads) {
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = lw_hash_value(seed, (uint64_t)keys[i]);
}

static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* Deduplicated R-MAT CSR (the C twin of device.generate_rmat_csr). off must hold
 * 2^scale+1 entries, col and val edge_factor*2^scale. Returns nnz (or -1). */
EXPORT int64_t lwo_rmat_csr(int scale, int64_t edge_factor, uint32_t ta, uint32_t tab,
                            uint32_t tabc, uint64_t seed, int threads, int64_t* off, int64_t* col,
                            double* val) {
    const int64_t n = (int64_t)1 << scale, n_edges = edge_factor * n;
    const int64_t mask = n - 1;
    int64_t* cursor = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_edges > 0 ? n_edges : 1));
    if (!cursor || !tmp) { free(cursor); free(tmp); return -1; }
    /* 1. row histogram */
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t e = 0; e < n_edges; ++e) {
        const int64_t r = (int64_t)(lw_rmat_key(seed, (uint64_t)e, scale, ta, tab, tabc) >> scale);
#pragma omp atomic
        cursor[r + 1] += 1;
    }
    for (int64_t r = 0; r < n; ++r) cursor[r + 1] += cursor[r];
    memcpy(off, cursor, sizeof(int64_t) * (size_t)(n + 1));
    /* 2. scatter columns by row (order inside a row fixed by the sort below) */
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t e = 0; e < n_edges; ++e) {
        const uint64_t k = lw_rmat_key(seed, (uint64_t)e, scale, ta, tab, tabc);
        const int64_t r = (int64_t)(k >> scale);
        int64_t pos;
#pragma omp atomic capture
        pos = cursor[r]++;
        tmp[pos] = (int64_t)(k & (uint64_t)mask);
    }
    /* 3. sort + unique every row; cursor[r] becomes the deduplicated length */
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4096)
    for (int64_t r = 0; r < n; ++r) {
        int64_t* c = tmp + off[r];
        const int64_t len = off[r + 1] - off[r];
        if (len > 1) qsort(c, (size_t)len, sizeof(int64_t), cmp_i64);
        int64_t u = 0;
        for (int64_t i = 0; i < len; ++i)
            if (i == 0 || c[i] != c[i - 1]) c[u++] = c[i];
        cursor[r] = u;
    }
    /* 4. compact into col, new offsets, hashed values */
    int64_t acc = 0;
    for (int64_t r = 0; r < n; ++r) {
        const int64_t len = cursor[r];
        cursor[r] = off[r];  /* old start */
        off[r] = acc;
        acc += len;
    }
    off[n] = acc;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 4096)
    for (int64_t r = 0; r < n; ++r) {
        const int64_t len = off[r + 1] - off[r];
        for (int64_t i = 0; i < len; ++i) {
            const int64_t c = tmp[cursor[r] + i];
            col[off[r] + i] = c;
            val[off[r] + i] = lw_hash_value(seed, ((uint64_t)r << scale) | (uint64_t)c);
        }
    }
    free(cursor);
    free(tmp);
    return acc;
}

/* ---- full-size checks on the device layout ---------------------------------
 * The same merge-path SpMV as lwo_spmv_merge_path (_fast.py:31-52 +
 * kernels.py:80-91), reading the GPU's arrays as they come back from the device:
 * offsets int32 or int64, columns int32, values and x float or double. Every
 * element is widened on load to int64 / fp64 — the reference's own coercion
 * (sparse.py:55-58, kernels.py:60) — so the arithmetic is the reference's, but a
 * 1e9-atom matrix needs no 16 GB upcast copy. scale[r] = sum_j |A_rj x_j| (the
 * north star's tolerance scale) comes out of the same pass, in the same lanes. */
#define LWO_NARROW_SPMV(NAME, OFF_T, VAL_T)                                                     \
    EXPORT int NAME(const OFF_T* off, const int32_t* col, const VAL_T* val, const VAL_T* x,      \
                    double* y, double* scale, int64_t rows, int64_t lanes, int threads) {       \
        const int64_t nnz = rows ? (int64_t)off[rows] : 0, total = rows + nnz;                  \
        const int64_t items = total ? (total + lanes - 1) / lanes : 0;                          \
        int64_t* coords = (int64_t*)malloc(sizeof(int64_t) * 2 * (size_t)(lanes + 1));          \
        int64_t* ct = (int64_t*)malloc(sizeof(int64_t) * (size_t)lanes);                        \
        double* cv = (double*)malloc(sizeof(double) * (size_t)lanes);                           \
        double* cs = (double*)malloc(sizeof(double) * (size_t)lanes);                           \
        if (!coords || !ct || !cv || !cs) {                                                      \
            free(coords); free(ct); free(cv); free(cs);                                          \
            return -1;                                                                           \
        }                                                                                        \
        _Pragma("omp parallel for num_threads(threads) schedule(static)")                        \
        for (int64_t k = 0; k <= lanes; ++k) {                                                   \
            const int64_t d = imin(k * items, total);                                            \
            int64_t lo = imax(0, d - nnz), hi = imin(d, rows);                                   \
            while (lo < hi) {                                                                    \
                const int64_t mid = (lo + hi + 1) / 2;                                           \
                if ((int64_t)off[mid] <= d - mid) lo = mid;                                      \
                else hi = mid - 1;                                                               \
            }                                                                                    \
            coords[2 * k] = lo;                                                                  \
            coords[2 * k + 1] = d - lo;                                                          \
        }                                                                                        \
        _Pragma("omp parallel for num_threads(threads) schedule(dynamic, 1)")                    \
        for (int64_t lane = 0; lane < lanes; ++lane) {                                           \
            int64_t atom = coords[2 * lane + 1];                                                 \
            const int64_t tile_end = coords[2 * lane + 2], atom_end = coords[2 * lane + 3];      \
            double acc = 0.0, sa = 0.0;                                                          \
            for (int64_t t = coords[2 * lane]; t < tile_end; ++t) {                              \
                for (; atom < (int64_t)off[t + 1]; ++atom) {                                     \
                    const double p = (double)val[atom] * (double)x[col[atom]];                   \
                    acc += p;                                                                    \
                    sa += p < 0 ? -p : p;                                                        \
                }                                                                                \
                y[t] = acc;                                                                      \
                scale[t] = sa;                                                                   \
                acc = 0.0;                                                                       \
                sa = 0.0;                                                                        \
            }                                                                                    \
            ct[lane] = -1;                                                                       \
            cv[lane] = 0.0;                                                                      \
            cs[lane] = 0.0;                                                                      \
            if (atom < atom_end) {                                                               \
                for (; atom < atom_end; ++atom) {                                                \
                    const double p = (double)val[atom] * (double)x[col[atom]];                   \
                    acc += p;                                                                    \
                    sa += p < 0 ? -p : p;                                                        \
                }                                                                                \
                ct[lane] = tile_end;                                                             \
                cv[lane] = acc;                                                                  \
                cs[lane] = sa;                                                                   \
            }                                                                                    \
        }                                                                                        \
        for (int64_t lane = 0; lane < lanes; ++lane)                                             \
            if (ct[lane] >= 0) {                                                                 \
                y[ct[lane]] += cv[lane];                                                         \
                scale[ct[lane]] += cs[lane];                                                     \
            }                                                                                    \
        free(coords); free(ct); free(cv); free(cs);                                              \
        return 0;                                                                                \
    }

LWO_NARROW_SPMV(lwo_spmv_narrow_o32_f32, int32_t, float)
LWO_NARROW_SPMV(lwo_spmv_narrow_o32_f64, int32_t, double)
LWO_NARROW_SPMV(lwo_spmv_narrow_o64_f32, int64_t, float)
LWO_NARROW_SPMV(lwo_spmv_narrow_o64_f64, int64_t, double)

/* max over rows of |y[r] - y_ref[r]| / (rtol * scale[r]) for a device result y
 * (float or double): the north star's per-entry bound as one number (<= 1 passes).
 * A row with scale 0 must match exactly (it holds only zero products). */
#define LWO_TOL(NAME, Y_T)                                                                      \
    EXPORT double NAME(const Y_T* y, const double* y_ref, const double* scale, int64_t rows,     \
                       double rtol, int64_t* worst_row, int threads) {                          \
        double worst = 0.0;                                                                      \
        int64_t wr = -1;                                                                         \
        _Pragma("omp parallel num_threads(threads)")                                             \
        {                                                                                        \
            double w = 0.0;                                                                      \
            int64_t r0 = -1;                                                                     \
            _Pragma("omp for schedule(static)")                                                  \
            for (int64_t r = 0; r < rows; ++r) {                                                 \
                const double e = fabs((double)y[r] - y_ref[r]);                                  \
                const double q = scale[r] > 0 ? e / (rtol * scale[r]) : (e > 0 ? INFINITY : 0.0); \
                if (q > w || q != q) { w = q != q ? INFINITY : q; r0 = r; }                      \
            }                                                                                    \
            _Pragma("omp critical")                                                              \
            if (w > worst || (w == worst && r0 >= 0 && (wr < 0 || r0 < wr))) { worst = w; wr = r0; } \
        }                                                                                        \
        if (worst_row) *worst_row = wr;                                                          \
        return worst;                                                                            \
    }

LWO_TOL(lwo_tolerance_f32, float)
LWO_TOL(lwo_tolerance_f64, double)
