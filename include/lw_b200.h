/*
 * lw_b200.h — C ABI of the B200-native load-balanced SpMV library (liblwb200.so).
 *
 * This is the drop-in boundary for the reference's compiled SpMV loops. The
 * reference (`lanework` 0.1.0, /root/reference/pkg/src/lanework) has no FFI: its
 * "plugin" seam is the backend switch in _backend.py:24-66 and the three numba
 * entry points in _fast.py that take raw arrays and return nothing. Every entry
 * point below names the reference interface it replaces.
 *
 * Conventions
 *   - Every pointer inside lw_csr_t / lw_probe_t and every x/y/workspace pointer
 *     is a DEVICE pointer owned by the caller (e.g. a torch CUDA tensor). The only
 *     exceptions are the *_host entry points, documented where they appear.
 *   - `stream` is a cudaStream_t passed as uintptr_t (0 = legacy default stream).
 *     All device entry points are stream-ordered and reentrant; none allocates
 *     memory behind the caller's back (workspace sizes come from *_workspace()).
 *   - Return value: 0 on success, otherwise a cudaError_t value (< 10000) or an
 *     LW_E_* code (>= 10000). lw_error_string() maps either to text.
 *   - Arithmetic: thread_mapped / group_mapped SpMV and every SpMM sum in fp64
 *     for fp32 and fp64 inputs; the work_oriented SpMV chunk scan adds at most
 *     IPT + 5 + NT/32 products in the value precision and carries partials across
 *     chunks and lanes in fp64. y is rounded to the input dtype once per row (plus
 *     once per carry fix-up for rows a work_oriented partition cuts).
 */
#ifndef LW_B200_H
#define LW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LW_ABI_VERSION 1

/* error codes (cudaError_t values pass through unchanged) */
#define LW_OK 0
#define LW_E_INVALID_ARG 10001   /* shape / config error: reference raises ValueError */
#define LW_E_UNSUPPORTED 10002   /* config the device kernels do not implement       */
#define LW_E_WORKSPACE 10003     /* workspace pointer NULL or smaller than required  */
#define LW_E_NO_DEVICE 10004     /* no CUDA device visible                           */
#define LW_E_FORMAT 10005        /* malformed input file: reference MatrixMarketError */

/* value dtypes */
#define LW_F32 0
#define LW_F64 1

/* schedules: values are the reference ScheduleKind members (schedules.py:21-24);
 * LW_WORK_ORIENTED is the north star's name for MERGE_PATH. */
#define LW_THREAD_MAPPED 0
#define LW_MERGE_PATH 1
#define LW_WORK_ORIENTED LW_MERGE_PATH
#define LW_GROUP_MAPPED 2

/* CSR operand. Mirrors reference CsrMatrix (sparse.py:40-71) with GPU storage:
 * row_offsets int32 or int64 (offset_bits), col_indices int32, values fp32/fp64. */
typedef struct lw_csr {
    int64_t rows;
    int64_t cols;
    int64_t nnz;
    const void* row_offsets;    /* [rows+1], int32 if offset_bits==32 else int64 */
    const int32_t* col_indices; /* [nnz] */
    const void* values;         /* [nnz], float if dtype==LW_F32 else double */
    int32_t offset_bits;        /* 32 | 64 */
    int32_t dtype;              /* LW_F32 | LW_F64 */
} lw_csr_t;

/* Optional instrumentation. Any field may be NULL. When the pointer passed to a
 * kernel entry point is non-NULL the instrumented kernel variant runs and records
 * exactly which lane processed which atom, attributed to which tile. This is the
 * GPU side of the reference's bit-exact schedule checks: lane_atoms must equal
 * executor.imbalance(ts, cfg).per_lane_atoms (executor.py:224-251), and
 * (atom_lane, atom_tile) must equal the (lane, tile) each atom receives from
 * execute_tile_major / execute_merge_path (executor.py:132-209). */
typedef struct lw_probe {
    int64_t* lane_atoms;  /* [lanes] atoms processed per lane; callee zeroes it */
    int32_t* atom_lane;   /* [nnz] lane that processed each atom               */
    int32_t* atom_tile;   /* [nnz] tile each atom was attributed to            */
    int32_t* atom_visits; /* [nnz] visit counter; caller zeroes it              */
} lw_probe_t;

/* Debug / introspection entry points over the probe: run the
 * instrumented SpMV of `schedule` (LW_THREAD_MAPPED / LW_MERGE_PATH /
 * LW_GROUP_MAPPED) into y and return per_lane_out[lanes] = atoms per lane
 * (executor.imbalance's per_lane_atoms), or atom_lane_out / atom_tile_out[nnz]
 * (the lane and tile of every atom, as execute_tile_major /
 * execute_merge_path assign them; either may be NULL). lanes = 0 selects
 * lw_auto_lanes(); the work_oriented schedule needs `workspace`
 * (lw_spmv_workspace). */
int lw_debug_lane_atom_counts(int schedule, const struct lw_csr* A, const void* x, void* y,
                              int64_t lanes, int64_t group_size, int64_t tiles_per_block,
                              int64_t* per_lane_out, void* workspace, size_t workspace_bytes,
                              uintptr_t stream);
int lw_debug_atom_tiles(int schedule, const struct lw_csr* A, const void* x, void* y, int64_t lanes,
                        int64_t group_size, int64_t tiles_per_block, int32_t* atom_lane_out,
                        int32_t* atom_tile_out, void* workspace, size_t workspace_bytes,
                        uintptr_t stream);

/* ---- library / device queries --------------------------------------------- */
const char* lw_error_string(int code);
int lw_abi_version(void);
/* SM count of the current device (cached per device). */
int lw_device_sm_count(int* sm_count_out);

/* Lane count P the device kernels pick when the caller leaves lanes at 0.
 * Replaces the reference default lanes = worker_threads*32 (executor.py:54-55)
 * with a device-sized value; group_size/tiles_per_block only matter for
 * LW_GROUP_MAPPED. */
int lw_auto_lanes(int schedule, int64_t rows, int64_t nnz, int64_t group_size,
                  int64_t tiles_per_block, int64_t* lanes_out);

/* ---- schedules ------------------------------------------------------------- */

/* Merge-path split points for `lanes` lanes over the (rows + nnz) path.
 * Replaces schedules.merge_path_partition (schedules.py:88-110) bit for bit:
 * coords[2k] = tile_k, coords[2k+1] = atom_k, k = 0..lanes, with
 * items = ceil((rows+nnz)/lanes) and diag_k = min(k*items, rows+nnz).
 * coords: device int64[(lanes+1)*2]. */
int lw_merge_path_partition(int64_t rows, int64_t nnz, const void* row_offsets,
                            int32_t offset_bits, int64_t lanes, int64_t* coords,
                            uintptr_t stream);

/* Group plan of every tile block: prefix[b*(tpb+1) + i] = exclusive prefix sum of
 * the atom counts of block b's tiles, computed with the same device scan the
 * group-mapped kernels use. Replaces schedules.group_plan(...).prefix
 * (schedules.py:137-159; exclusive_prefix_sum 121-130); short last block is
 * padded with its total. prefix: device int64[nblocks*(tpb+1)]. */
int lw_group_plan_prefix(int64_t rows, const void* row_offsets, int32_t offset_bits,
                         int64_t tiles_per_block, int64_t* prefix, uintptr_t stream);

/* ---- SpMV: y = A x, one kernel family per schedule ------------------------- */

/* thread_mapped: lane l owns tiles l, l+P, ... and assigns y[t].
 * Replaces _fast.spmv_thread_mapped (_fast.py:20-28) + its run_sharded fan-out
 * (kernels.py:74-79). lanes = 0 selects lw_auto_lanes(). */
int lw_spmv_thread_mapped(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                          const lw_probe_t* probe, uintptr_t stream);

/* work_oriented (merge-path): even share of rows+nnz per lane, carries fixed up
 * in lane order on the device. Replaces _fast.spmv_merge_path (_fast.py:31-52)
 * plus the host partition (kernels.py:81) and the serial carry fix-up
 * (kernels.py:90-91). lanes = 0 selects lw_auto_lanes(). The SpMV and fix-up
 * kernels are programmatic dependent launches of the kernel before them (they
 * wait for its results on the device); to the caller the call is ordinary
 * stream-ordered work: it starts after everything queued before it and
 * everything queued after it sees its y. */
size_t lw_spmv_work_oriented_workspace(int64_t rows, int64_t nnz, int64_t lanes,
                                       int32_t dtype);
int lw_spmv_work_oriented(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                          void* workspace, size_t workspace_bytes,
                          const lw_probe_t* probe, uintptr_t stream);
/* The same call split into its three stream-ordered phases so a caller can
 * bracket each with events: bit 0 = merge-path partition, bit 1 = even-share
 * SpMV kernel, bit 2 = carry fix-up. Running 1, then 2, then 4 on one stream
 * equals lw_spmv_work_oriented(..., probe = NULL). */
int lw_spmv_work_oriented_phases(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                                 void* workspace, size_t workspace_bytes,
                                 uint32_t phase_mask, uintptr_t stream);

/* Hot-x column packing: an inspector-executor form of the
 * work_oriented SpMV for power-law matrices. No reference counterpart — it is a
 * B200 layout step in front of lw_spmv_work_oriented; y is bit-identical.
 * lw_hotx_build (one-time, per matrix; synchronizes `stream`, reads two 256 KB
 * histograms on the host): picks the hot set H = {c : count(c) >= T}, T the
 * smallest threshold >= 2 with |H| <= max_hot (<= 32768), writes hot_cols[|H|]
 * (ascending) and col_packed[nnz] (hot columns -> slot | 0x80000000), *n_hot_out
 * = |H|. lw_spmv_work_oriented_hotx: A's col_indices must be col_packed; packs
 * xh[s] = x[hot_cols[s]] into the workspace, then runs the work_oriented SpMV
 * with hot gathers kept in L1 and cold ones bypassing it. */
/* Symmetric permutation P A P^T of a square CSR (degree relabeling for the
 * iterated SpMV, C5): output row i is input row order[i] with every column c
 * renamed rank[c] (rank = order^-1, device int32[cols]; order device
 * int64[rows]); atoms keep their order inside a row. off_out (rows+1 entries,
 * the input's offset width) is the caller's prefix sum of the permuted row
 * lengths; col_out / val_out hold nnz entries. One-time inspector step; no
 * reference counterpart (the reference iterates in the input numbering). */
int lw_csr_permute(const lw_csr_t* A, const int64_t* order, const int32_t* rank, const void* off_out,
                   int32_t* col_out, void* val_out, uintptr_t stream);

size_t lw_hotx_build_workspace(int64_t cols);
int lw_hotx_build(const lw_csr_t* A, int32_t max_hot, int32_t* col_packed, int32_t* hot_cols,
                  int32_t* n_hot_out, void* workspace, size_t workspace_bytes, uintptr_t stream);
size_t lw_spmv_work_oriented_hotx_workspace(int64_t rows, int64_t nnz, int64_t lanes,
                                            int32_t n_hot, int32_t dtype);
int lw_spmv_work_oriented_hotx(const lw_csr_t* A_packed, const int32_t* hot_cols, int32_t n_hot,
                               const void* x, void* y, int64_t lanes, void* workspace,
                               size_t workspace_bytes, uintptr_t stream);

/* The same in three stream-ordered phases (bit 0: partition + pack of x into the
 * workspace's hot slots, one launch; bit 1: SpMV chunk kernel; bit 2: carry
 * fix-up), as lw_spmv_work_oriented_phases; phases 1 and 2 must see the same x. */
int lw_spmv_work_oriented_hotx_phases(const lw_csr_t* A_packed, const int32_t* hot_cols,
                                      int32_t n_hot, const void* x, void* y, int64_t lanes,
                                      void* workspace, size_t workspace_bytes,
                                      uint32_t phase_mask, uintptr_t stream);

/* work_oriented SpMV fused with the all-gather of the power iteration (BASELINE
 * C5): every row this rank's shard produces is written to y AND to
 * element row_base + row of each rank's next-x buffer -- through the NVLS
 * multicast address (multimem.st, one store reaches every GPU) when
 * multicast_ptr != 0, else one peer-to-peer store per buffer in peer_ptrs
 * (n_peers <= 8, HOST array of device addresses, e.g. symmetric-memory
 * buffer_ptrs). Rows a lane boundary cuts are rewritten with their final value
 * by the carry fix-up, so after a cross-GPU barrier every buffer holds the full
 * y. Replaces SpMV + NCCL all-gather with one pass over NVLink. */
int lw_spmv_work_oriented_peers(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                                void* workspace, size_t workspace_bytes, int32_t n_peers,
                                const uint64_t* peer_ptrs, uint64_t multicast_ptr,
                                int64_t row_base, uintptr_t stream);
/* The same over a hot-x packed matrix (lw_hotx_build): A_packed/hot_cols/n_hot
 * as for lw_spmv_work_oriented_hotx; workspace lw_spmv_work_oriented_hotx_workspace. */
int lw_spmv_work_oriented_peers_hotx(const lw_csr_t* A_packed, const int32_t* hot_cols,
                                     int32_t n_hot, const void* x, void* y, int64_t lanes,
                                     void* workspace, size_t workspace_bytes, int32_t n_peers,
                                     const uint64_t* peer_ptrs, uint64_t multicast_ptr,
                                     int64_t row_base, uintptr_t stream);

/* Power-iteration normalisation (BASELINE C5; the reference driver's x = y/||y||):
 * lw_vector_norm writes ||y||_2 (fp64, deterministic two-level reduction) to the
 * DEVICE scalar norm_out; lw_vector_scale writes x = y / norm (x = y when the
 * norm is 0) reading the device scalar, so the pair runs without a host sync;
 * x may equal y (in-place).
 * Workspace: lw_norm_workspace(n) bytes of device memory. */
size_t lw_norm_workspace(int64_t n);
int lw_vector_norm(const void* y, int64_t n, int32_t dtype, void* workspace,
                   size_t workspace_bytes, double* norm_out, uintptr_t stream);
int lw_vector_scale(const void* y, int64_t n, int32_t dtype, const double* norm, void* x_out,
                    uintptr_t stream);

/* group_mapped: groups of group_size lanes own blocks of tiles_per_block tiles,
 * members take block atoms by member stride (schedules.py:137-167,
 * executor.py:149-168). Replaces _fast.spmv_group_mapped (_fast.py:55-77).
 * (32,32) runs the warp-tile kernel, (B,B) for B in {64,128,256} the block-tile
 * kernel, anything else the general group kernel. lanes = 0 selects auto. */
int lw_spmv_group_mapped(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                         int64_t group_size, int64_t tiles_per_block,
                         const lw_probe_t* probe, uintptr_t stream);

/* Schedule-dispatching form of the three calls above (the shape of the
 * reference operator kernels.spmv, kernels.py:57-69). workspace is only used by
 * LW_MERGE_PATH; size it with lw_spmv_workspace(). */
size_t lw_spmv_workspace(int schedule, int64_t rows, int64_t nnz, int64_t lanes,
                         int32_t dtype);
int lw_spmv(int schedule, const lw_csr_t* A, const void* x, void* y, int64_t lanes,
            int64_t group_size, int64_t tiles_per_block, void* workspace,
            size_t workspace_bytes, uintptr_t stream);

/* Host-buffer form for FFI callers that hold NumPy/host arrays (the ctypes
 * binding in INTEGRATION.md). A's pointers, x and y are HOST pointers (pinned
 * or pageable); the call allocates device buffers stream-ordered, copies in,
 * runs lw_spmv, copies y out and synchronizes `stream` before returning. */
int lw_spmv_host(int schedule, const lw_csr_t* A_host, const void* x_host, void* y_host,
                 int64_t lanes, int64_t group_size, int64_t tiles_per_block,
                 uintptr_t stream);

/* ---- SpMM: C = A B, B dense row-major [cols x n], C row-major [rows x n] ---------
 * The column loop wrapped around the SpMV body (Listing 4). Replaces
 * kernels.spmm (kernels.py:129-175) and _fast.spmm_{thread_mapped,merge_path,
 * group_mapped} (_fast.py:80-144): same schedules (a lane owns the same tiles and
 * atoms as in SpMV), each atom adding val * B[col, :] to its row. A lane is a
 * team of threads covering up to 32x16 bytes of columns; wider n is walked in
 * slabs. B and C are device pointers; 16-byte aligned B/C with n a multiple of
 * 4 (fp32) / 2 (fp64) take the vector path. lanes = 0 selects
 * lw_spmm_auto_lanes(). Sums are fp64; group_mapped sums each C[tile, :] in the
 * reference's member-major C += v * B[src] order (no atomics; bit-identical to
 * the reference for fp64 data). */
int lw_spmm_auto_lanes(int schedule, int64_t rows, int64_t nnz, int64_t n, int64_t group_size,
                       int64_t tiles_per_block, int64_t* lanes_out);
size_t lw_spmm_workspace(int schedule, int64_t rows, int64_t nnz, int64_t n, int64_t lanes,
                         int32_t dtype);
int lw_spmm_thread_mapped(const lw_csr_t* A, const void* B, void* C, int64_t n, int64_t lanes,
                          uintptr_t stream);
int lw_spmm_work_oriented(const lw_csr_t* A, const void* B, void* C, int64_t n, int64_t lanes,
                          void* workspace, size_t workspace_bytes, uintptr_t stream);
int lw_spmm_group_mapped(const lw_csr_t* A, const void* B, void* C, int64_t n, int64_t lanes,
                         int64_t group_size, int64_t tiles_per_block, uintptr_t stream);
int lw_spmm(int schedule, const lw_csr_t* A, const void* B, void* C, int64_t n, int64_t lanes,
            int64_t group_size, int64_t tiles_per_block, void* workspace, size_t workspace_bytes,
            uintptr_t stream);

/* ---- SSSP / BFS: frontier relaxation under the three schedules ---------------
 * Replaces kernels.sssp / sssp_pass / bfs (kernels.py:230-381) and the numba
 * relax loops (_fast.py:147-170); the paper's Listing 5. G is a square CSR
 * (row = source vertex, value = non-negative edge weight, fp32 or fp64). A pass
 * takes the compacted frontier active[n_active] (vertex ids in increasing order,
 * = np.flatnonzero(in_frontier)), builds the frontier tile set (tiles = active
 * vertices, atoms = out-edges) on the device and relaxes every atom under the
 * schedule: SSSP by atomicMin on the fp64 bit pattern of dist (out[v] = 1 when
 * the distance strictly improved), BFS by claiming depth[v] < 0 with next_depth.
 * out_frontier is zeroed by the pass. dist is fp64 (+inf unreached), depth
 * int64 (-1 = UNREACHED). lw_sssp / lw_bfs run the whole traversal (one host
 * synchronization per pass for the frontier size) and report the pass count.
 * Workspace: lw_frontier_workspace(rows) bytes of device memory. */
size_t lw_frontier_workspace(int64_t n_vertices);
int lw_frontier_compact(const uint8_t* mask, int64_t n, int32_t* active, int64_t* count_dev,
                        void* workspace, size_t workspace_bytes, uintptr_t stream);
int lw_sssp_pass(const lw_csr_t* G, const int32_t* active, int64_t n_active, double* dist,
                 uint8_t* out_frontier, int schedule, int64_t lanes, int64_t group_size,
                 int64_t tiles_per_block, void* workspace, size_t workspace_bytes,
                 uintptr_t stream);
int lw_bfs_pass(const lw_csr_t* G, const int32_t* active, int64_t n_active, int64_t* depth,
                int64_t next_depth, uint8_t* out_frontier, int schedule, int64_t lanes,
                int64_t group_size, int64_t tiles_per_block, void* workspace,
                size_t workspace_bytes, uintptr_t stream);
int lw_sssp(const lw_csr_t* G, int64_t source, double* dist, int schedule, int64_t lanes,
            int64_t group_size, int64_t tiles_per_block, void* workspace, size_t workspace_bytes,
            int64_t* passes_out, uintptr_t stream);
int lw_bfs(const lw_csr_t* G, int64_t source, int64_t* depth, int schedule, int64_t lanes,
           int64_t group_size, int64_t tiles_per_block, void* workspace, size_t workspace_bytes,
           int64_t* passes_out, uintptr_t stream);

/* ---- ingestion (host-native; the input side of the path) ---------------------
 * Matrix Market coordinate text -> COO -> CSR. Replaces mmio.parse_matrix_market
 * (mmio.py:24-107) and sparse.coo_to_csr (sparse.py:130-150). Buffers are HOST
 * memory. Parsing is multi-threaded over line-aligned chunks; accepted syntax,
 * error precedence (first bad line in file order) and messages follow mmio.py,
 * returned as LW_E_FORMAT with the text in err[errlen]. */
typedef struct lw_mm_header {
    int64_t rows;
    int64_t cols;
    int64_t entries;     /* declared entry count */
    int32_t field;       /* 0 real, 1 integer, 2 pattern */
    int32_t symmetric;   /* 0 general, 1 symmetric (mirrored entries appended) */
    int64_t data_offset; /* byte offset of the first line after the size header */
} lw_mm_header_t;

int lw_mm_parse_header(const char* buf, size_t len, lw_mm_header_t* header, char* err,
                       size_t errlen);
/* row/col/val hold capacity >= entries (x2 when symmetric) entries; *count_out
 * receives the COO entry count (stored + mirrored off-diagonal). threads <= 0:
 * all hardware threads. Indices are 0-based, pattern values 1.0. */
int lw_mm_parse_entries(const char* buf, size_t len, const lw_mm_header_t* header, int64_t* row,
                        int64_t* col, double* val, int64_t capacity, int64_t* count_out,
                        int32_t threads, char* err, size_t errlen);
/* Sort by (row, col), sum duplicates in input order (as np.bincount does),
 * pack CSR: row_offsets[rows+1], col_out/val_out[>= n]; *nnz_out distinct
 * pairs. LW_E_INVALID_ARG on an out-of-bounds entry. */
int lw_coo_to_csr_host(int64_t rows, int64_t cols, int64_t n, const int64_t* row,
                       const int64_t* col, const double* val, int64_t* row_offsets,
                       int64_t* col_out, double* val_out, int64_t* nnz_out, int32_t threads);

/* ---- synthetic inputs (counter-based, identical on host oracle and device) ---- */

/* R-MAT edge keys: keys[i] = (row << scale) | col of edge e = edge_begin + i,
 * i in [0, n_edges) (chunked generation of one edge stream), each
 * of the `scale` levels choosing a quadrant with 32-bit thresholds
 * t_a < t_ab < t_abc (a, a+b, a+b+c scaled by 2^32). keys: device int64. */
int lw_rmat_keys(int32_t scale, int64_t edge_begin, int64_t n_edges, uint32_t t_a, uint32_t t_ab,
                 uint32_t t_abc, uint64_t seed, int64_t* keys, uintptr_t stream);

/* Uniform keys: keys[i] = lw_uniform_key(seed, begin + i, space) in [0, space)
 * (row * cols + col for a rows x cols matrix; sorted + deduplicated by the
 * caller). Feeds the uniform-random configs (C2u, C4 uniform) at sizes the
 * reference's host generator (sparse.py:164-187) takes minutes to build. */
int lw_uniform_keys(int64_t space, int64_t begin, int64_t n, uint64_t seed, int64_t* keys,
                    uintptr_t stream);

/* values[i] = U[-1,1) drawn from hash(seed, key[i]); dtype LW_F32 rounds the fp64
 * draw to fp32. */
int lw_hash_values(const int64_t* keys, int64_t n, uint64_t seed, int32_t dtype,
                   void* values, uintptr_t stream);

#ifdef __cplusplus
}
#endif

#endif /* LW_B200_H */
