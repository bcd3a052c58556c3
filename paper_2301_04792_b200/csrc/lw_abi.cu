// lw_abi.cu — extern "C" entry points of liblwb200.so (declared in include/lw_b200.h).
// Argument validation mirrors the reference's ValueError cases (kernels.py:61-62,
// executor.py:51-63): bad shapes/configs return LW_E_INVALID_ARG, never abort.
#include <cstring>
#include <mutex>

#include "lw_common.cuh"

namespace lw {
int spmv_thread_mapped(const lw_csr_t*, const void*, void*, int64_t, const lw_probe_t*, cudaStream_t);
int spmv_work_oriented(const lw_csr_t*, const void*, void*, int64_t, void*, size_t, const lw_probe_t*, unsigned, cudaStream_t);
int spmv_group_mapped(const lw_csr_t*, const void*, void*, int64_t, int64_t, int64_t, const lw_probe_t*, cudaStream_t);
size_t wo_workspace(int64_t rows, int64_t nnz, int64_t lanes, int dtype);
int64_t wo_lanes(int64_t rows, int64_t nnz, int64_t lanes);
int64_t group_auto_lanes(int64_t rows, int64_t gs, int64_t tpb);
int merge_path_partition(int64_t, int64_t, const void*, int, int64_t, int64_t*, cudaStream_t);
int group_plan_prefix(int64_t, const void*, int, int64_t, int64_t*, cudaStream_t);
int rmat_keys(int, int64_t, int64_t, uint32_t, uint32_t, uint32_t, uint64_t, int64_t*, cudaStream_t);
int hash_values(const int64_t*, int64_t, uint64_t, int, void*, cudaStream_t);
int uniform_keys(int64_t, int64_t, int64_t, uint64_t, int64_t*, cudaStream_t);
int spmm(int, const lw_csr_t*, const void*, void*, int64_t, int64_t, int64_t, int64_t, void*, size_t, cudaStream_t);
int64_t spmm_auto_lanes(int schedule, int64_t rows, int64_t nnz, int64_t n, int64_t gs, int64_t tpb);
size_t spmm_wo_workspace(int64_t lanes, int64_t n);
size_t frontier_workspace(int64_t n);
size_t norm_workspace(int64_t n);
int vector_norm(const void*, int64_t, int, void*, double*, cudaStream_t);
int vector_scale(const void*, int64_t, int, const double*, void*, cudaStream_t);
int spmv_work_oriented_peers(const lw_csr_t*, const void*, void*, int64_t, void*, size_t, int32_t,
                             const uint64_t*, uint64_t, int64_t, cudaStream_t, const int32_t*, int32_t);
size_t wo_hotx_workspace(int64_t rows, int64_t nnz, int64_t lanes, int64_t n_hot, int dtype);
int spmv_work_oriented_hotx(const lw_csr_t*, const int32_t*, int32_t, const void*, void*, int64_t, void*,
                            size_t, unsigned, cudaStream_t);
size_t hotx_build_workspace(int64_t cols);
int csr_permute(const lw_csr_t*, const int64_t*, const int32_t*, const void*, int32_t*, void*, cudaStream_t);
int hotx_build(const lw_csr_t*, int32_t, int32_t*, int32_t*, int32_t*, void*, size_t, cudaStream_t);
int frontier_compact(const uint8_t*, int64_t, int32_t*, int64_t*, void*, cudaStream_t);
int sssp_pass(const lw_csr_t*, const int32_t*, int64_t, double*, uint8_t*, int, int64_t, int64_t, int64_t, void*, cudaStream_t);
int bfs_pass(const lw_csr_t*, const int32_t*, int64_t, int64_t*, int64_t, uint8_t*, int, int64_t, int64_t, int64_t, void*, cudaStream_t);
int sssp_run(const lw_csr_t*, int64_t, double*, int, int64_t, int64_t, int64_t, void*, int64_t*, cudaStream_t);
int bfs_run(const lw_csr_t*, int64_t, int64_t*, int, int64_t, int64_t, int64_t, void*, int64_t*, cudaStream_t);

static int g_sm[64];
static std::mutex g_sm_mu;

int sm_count() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    std::lock_guard<std::mutex> lk(g_sm_mu);
    if (!g_sm[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
        g_sm[dev] = n;
    }
    return g_sm[dev];
}

static int64_t thread_auto_lanes(int64_t rows) {
    const int64_t cap = (int64_t)sm_count() * 2048;
    int64_t p = ceil_div(rows > 0 ? rows : 1, 256) * 256;
    return p < cap ? p : cap;
}

static int check_csr(const lw_csr_t* A) {
    if (!A) return LW_E_INVALID_ARG;
    if (A->rows < 0 || A->cols < 0 || A->nnz < 0) return LW_E_INVALID_ARG;
    if (A->offset_bits != 32 && A->offset_bits != 64) return LW_E_INVALID_ARG;
    if (A->dtype != LW_F32 && A->dtype != LW_F64) return LW_E_INVALID_ARG;
    if (A->offset_bits == 32 && A->nnz > 0x7fffffffLL) return LW_E_INVALID_ARG;
    if (A->rows > 0 && !A->row_offsets) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && (!A->col_indices || !A->values)) return LW_E_INVALID_ARG;
    return LW_OK;
}

static int resolve_lanes(int schedule, const lw_csr_t* A, int64_t lanes, int64_t gs, int64_t tpb,
                         int64_t* out) {
    if (lanes < 0) return LW_E_INVALID_ARG;
    if (lanes > 0) { *out = lanes; return LW_OK; }
    switch (schedule) {
        case LW_THREAD_MAPPED: *out = thread_auto_lanes(A->rows); return LW_OK;
        case LW_MERGE_PATH: *out = wo_lanes(A->rows, A->nnz, 0); return LW_OK;
        case LW_GROUP_MAPPED:
            if (gs < 1 || tpb < 1) return LW_E_INVALID_ARG;
            *out = group_auto_lanes(A->rows, gs, tpb);
            return LW_OK;
        default: return LW_E_INVALID_ARG;
    }
}

}  // namespace lw

using namespace lw;

extern "C" {

const char* lw_error_string(int code) {
    switch (code) {
        case LW_OK: return "success";
        case LW_E_INVALID_ARG: return "invalid argument (shape or schedule configuration)";
        case LW_E_UNSUPPORTED: return "configuration not supported by the device kernels";
        case LW_E_WORKSPACE: return "workspace missing or smaller than required";
        case LW_E_NO_DEVICE: return "no CUDA device visible";
        case LW_E_FORMAT: return "malformed input file";
        default: return cudaGetErrorString((cudaError_t)code);
    }
}

int lw_abi_version(void) { return LW_ABI_VERSION; }

int lw_device_sm_count(int* out) {
    if (!out) return LW_E_INVALID_ARG;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return LW_E_NO_DEVICE;
    *out = sm_count();
    return LW_OK;
}

int lw_auto_lanes(int schedule, int64_t rows, int64_t nnz, int64_t gs, int64_t tpb,
                  int64_t* lanes_out) {
    if (!lanes_out || rows < 0 || nnz < 0) return LW_E_INVALID_ARG;
    lw_csr_t a{};
    a.rows = rows;
    a.nnz = nnz;
    return resolve_lanes(schedule, &a, 0, gs, tpb, lanes_out);
}

int lw_merge_path_partition(int64_t rows, int64_t nnz, const void* off, int32_t bits,
                            int64_t lanes, int64_t* coords, uintptr_t stream) {
    if (bits != 32 && bits != 64) return LW_E_INVALID_ARG;
    return merge_path_partition(rows, nnz, off, bits, lanes, coords, (cudaStream_t)stream);
}

int lw_group_plan_prefix(int64_t rows, const void* off, int32_t bits, int64_t tpb,
                         int64_t* prefix, uintptr_t stream) {
    if (bits != 32 && bits != 64) return LW_E_INVALID_ARG;
    return group_plan_prefix(rows, off, bits, tpb, prefix, (cudaStream_t)stream);
}

int lw_spmv_thread_mapped(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                          const lw_probe_t* probe, uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    if (A->rows > 0 && !y) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && !x) return LW_E_INVALID_ARG;
    int64_t p = 0;
    if ((rc = resolve_lanes(LW_THREAD_MAPPED, A, lanes, 0, 0, &p))) return rc;
    return spmv_thread_mapped(A, x, y, p, probe, (cudaStream_t)stream);
}

size_t lw_spmv_work_oriented_workspace(int64_t rows, int64_t nnz, int64_t lanes, int32_t dtype) {
    if (rows < 0 || nnz < 0 || lanes < 0 || (dtype != LW_F32 && dtype != LW_F64)) return 0;
    return wo_workspace(rows, nnz, lanes, dtype);   // fp64 lanes hold more (smaller) chunks
}

int lw_spmv_work_oriented(const lw_csr_t* A, const void* x, void* y, int64_t lanes, void* ws,
                          size_t ws_bytes, const lw_probe_t* probe, uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    if (A->rows > 0 && !y) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && !x) return LW_E_INVALID_ARG;
    if (lanes < 0) return LW_E_INVALID_ARG;
    return spmv_work_oriented(A, x, y, lanes, ws, ws_bytes, probe, 7u, (cudaStream_t)stream);
}

int lw_spmv_work_oriented_phases(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                                 void* ws, size_t ws_bytes, uint32_t phase_mask,
                                 uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    if (A->rows > 0 && !y) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && !x) return LW_E_INVALID_ARG;
    if (lanes < 0 || phase_mask == 0 || phase_mask > 7u) return LW_E_INVALID_ARG;
    return spmv_work_oriented(A, x, y, lanes, ws, ws_bytes, nullptr, phase_mask, (cudaStream_t)stream);
}

int lw_spmv_work_oriented_peers(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                                void* ws, size_t ws_bytes, int32_t n_peers,
                                const uint64_t* peer_ptrs, uint64_t multicast_ptr,
                                int64_t row_base, uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    if (A->rows > 0 && !y) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && !x) return LW_E_INVALID_ARG;
    if (lanes < 0 || (n_peers == 0 && multicast_ptr == 0)) return LW_E_INVALID_ARG;
    return spmv_work_oriented_peers(A, x, y, lanes, ws, ws_bytes, n_peers, peer_ptrs, multicast_ptr,
                                    row_base, (cudaStream_t)stream, nullptr, 0);
}

int lw_spmv_work_oriented_peers_hotx(const lw_csr_t* A, const int32_t* hot_cols, int32_t n_hot,
                                     const void* x, void* y, int64_t lanes, void* ws,
                                     size_t ws_bytes, int32_t n_peers, const uint64_t* peer_ptrs,
                                     uint64_t multicast_ptr, int64_t row_base, uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    if (A->rows > 0 && !y) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && !x) return LW_E_INVALID_ARG;
    if (lanes < 0 || (n_peers == 0 && multicast_ptr == 0)) return LW_E_INVALID_ARG;
    static const int32_t none = 0;   // selects the packed kernel even with no hot slots
    return spmv_work_oriented_peers(A, x, y, lanes, ws, ws_bytes, n_peers, peer_ptrs, multicast_ptr,
                                    row_base, (cudaStream_t)stream, hot_cols ? hot_cols : &none, n_hot);
}

int lw_csr_permute(const lw_csr_t* A, const int64_t* order, const int32_t* rank, const void* off_out,
                   int32_t* col_out, void* val_out, uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    return csr_permute(A, order, rank, off_out, col_out, val_out, (cudaStream_t)stream);
}

size_t lw_hotx_build_workspace(int64_t cols) { return cols < 0 ? 0 : hotx_build_workspace(cols); }

int lw_hotx_build(const lw_csr_t* A, int32_t max_hot, int32_t* col_packed, int32_t* hot_cols,
                  int32_t* n_hot_out, void* ws, size_t ws_bytes, uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    return hotx_build(A, max_hot, col_packed, hot_cols, n_hot_out, ws, ws_bytes, (cudaStream_t)stream);
}

size_t lw_spmv_work_oriented_hotx_workspace(int64_t rows, int64_t nnz, int64_t lanes, int32_t n_hot,
                                            int32_t dtype) {
    if (rows < 0 || nnz < 0 || lanes < 0 || n_hot < 0) return 0;
    return wo_hotx_workspace(rows, nnz, lanes, n_hot, dtype);
}

int lw_spmv_work_oriented_hotx(const lw_csr_t* A, const int32_t* hot_cols, int32_t n_hot,
                               const void* x, void* y, int64_t lanes, void* ws, size_t ws_bytes,
                               uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    if (A->rows > 0 && !y) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && !x) return LW_E_INVALID_ARG;
    if (lanes < 0) return LW_E_INVALID_ARG;
    return spmv_work_oriented_hotx(A, hot_cols, n_hot, x, y, lanes, ws, ws_bytes, 7u, (cudaStream_t)stream);
}

int lw_spmv_work_oriented_hotx_phases(const lw_csr_t* A, const int32_t* hot_cols, int32_t n_hot,
                                      const void* x, void* y, int64_t lanes, void* ws,
                                      size_t ws_bytes, uint32_t phase_mask, uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    if (A->rows > 0 && !y) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && !x) return LW_E_INVALID_ARG;
    if (lanes < 0 || phase_mask == 0 || phase_mask > 7u) return LW_E_INVALID_ARG;
    return spmv_work_oriented_hotx(A, hot_cols, n_hot, x, y, lanes, ws, ws_bytes, phase_mask,
                                   (cudaStream_t)stream);
}

int lw_spmv_group_mapped(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                         int64_t gs, int64_t tpb, const lw_probe_t* probe, uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    if (A->rows > 0 && !y) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && !x) return LW_E_INVALID_ARG;
    if (gs < 1 || tpb < 1) return LW_E_INVALID_ARG;
    int64_t p = 0;
    if ((rc = resolve_lanes(LW_GROUP_MAPPED, A, lanes, gs, tpb, &p))) return rc;
    return spmv_group_mapped(A, x, y, p, gs, tpb, probe, (cudaStream_t)stream);
}

// ---- debug / introspection over the probe ----------------------------
static int debug_probe_run(int schedule, const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                           int64_t gs, int64_t tpb, const lw_probe_t* pr, void* ws, size_t ws_bytes,
                           uintptr_t stream) {
    switch (schedule) {
        case LW_THREAD_MAPPED: return lw_spmv_thread_mapped(A, x, y, lanes, pr, stream);
        case LW_MERGE_PATH: return lw_spmv_work_oriented(A, x, y, lanes, ws, ws_bytes, pr, stream);
        case LW_GROUP_MAPPED: return lw_spmv_group_mapped(A, x, y, lanes, gs, tpb, pr, stream);
        default: return LW_E_INVALID_ARG;
    }
}

int lw_debug_lane_atom_counts(int schedule, const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                              int64_t gs, int64_t tpb, int64_t* per_lane_out, void* ws, size_t ws_bytes,
                              uintptr_t stream) {
    if (!per_lane_out) return LW_E_INVALID_ARG;
    lw_probe_t pr{per_lane_out, nullptr, nullptr, nullptr};
    return debug_probe_run(schedule, A, x, y, lanes, gs, tpb, &pr, ws, ws_bytes, stream);
}

int lw_debug_atom_tiles(int schedule, const lw_csr_t* A, const void* x, void* y, int64_t lanes, int64_t gs,
                        int64_t tpb, int32_t* atom_lane_out, int32_t* atom_tile_out, void* ws, size_t ws_bytes,
                        uintptr_t stream) {
    if (!atom_lane_out && !atom_tile_out) return LW_E_INVALID_ARG;
    lw_probe_t pr{nullptr, atom_lane_out, atom_tile_out, nullptr};
    return debug_probe_run(schedule, A, x, y, lanes, gs, tpb, &pr, ws, ws_bytes, stream);
}

size_t lw_spmv_workspace(int schedule, int64_t rows, int64_t nnz, int64_t lanes, int32_t dtype) {
    return schedule == LW_MERGE_PATH ? lw_spmv_work_oriented_workspace(rows, nnz, lanes, dtype) : 0;
}

int lw_spmv(int schedule, const lw_csr_t* A, const void* x, void* y, int64_t lanes, int64_t gs,
            int64_t tpb, void* ws, size_t ws_bytes, uintptr_t stream) {
    switch (schedule) {
        case LW_THREAD_MAPPED: return lw_spmv_thread_mapped(A, x, y, lanes, nullptr, stream);
        case LW_MERGE_PATH: return lw_spmv_work_oriented(A, x, y, lanes, ws, ws_bytes, nullptr, stream);
        case LW_GROUP_MAPPED: return lw_spmv_group_mapped(A, x, y, lanes, gs, tpb, nullptr, stream);
        default: return LW_E_INVALID_ARG;
    }
}

// lw_spmv_host's device staging comes from a private stream-ordered pool per
// device, created once and told to keep its freed memory mapped (re-mapping GBs
// on every call would dominate it). Private, so the caller's default pool and
// any other cudaMallocAsync user in the process keep their own release policy.
static int staging_pool(cudaMemPool_t* out) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    LW_TRY(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) return LW_E_UNSUPPORTED;
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
        cudaMemPoolProps props = {};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p;
        LW_TRY(cudaMemPoolCreate(&p, &props));
        uint64_t keep = UINT64_MAX;
        LW_TRY(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep));
        pools[dev] = p;
    }
    *out = pools[dev];
    return LW_OK;
}

int lw_spmv_host(int schedule, const lw_csr_t* H, const void* x_host, void* y_host, int64_t lanes,
                 int64_t gs, int64_t tpb, uintptr_t stream) {
    int rc = check_csr(H);
    if (rc) return rc;
    if (H->rows > 0 && !y_host) return LW_E_INVALID_ARG;
    if (H->cols > 0 && !x_host) return LW_E_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t vb = H->dtype == LW_F32 ? 4 : 8, ob = H->offset_bits / 8;
    const size_t off_b = (size_t)(H->rows + 1) * ob, col_b = (size_t)H->nnz * 4,
                 val_b = (size_t)H->nnz * vb, x_b = (size_t)H->cols * vb, y_b = (size_t)H->rows * vb;
    const size_t ws_b = lw_spmv_workspace(schedule, H->rows, H->nnz, lanes, H->dtype);
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t bytes = up(off_b) + up(col_b) + up(val_b) + up(x_b) + up(y_b) + up(ws_b);
    unsigned char* d = nullptr;
    cudaMemPool_t pool;
    if ((rc = staging_pool(&pool))) return rc;
    LW_TRY(cudaMallocFromPoolAsync((void**)&d, bytes > 0 ? bytes : 256, pool, s));
    unsigned char* p = d;
    void* d_off = p; p += up(off_b);
    void* d_col = p; p += up(col_b);
    void* d_val = p; p += up(val_b);
    void* d_x = p;   p += up(x_b);
    void* d_y = p;   p += up(y_b);
    void* d_ws = p;
    rc = LW_OK;
    auto cp = [&](void* dst, const void* src, size_t b) {
        if (!rc && b) rc = (int)cudaMemcpyAsync(dst, src, b, cudaMemcpyHostToDevice, s);
    };
    cp(d_off, H->row_offsets, off_b);
    cp(d_col, H->col_indices, col_b);
    cp(d_val, H->values, val_b);
    cp(d_x, x_host, x_b);
    if (!rc) {
        lw_csr_t A = *H;
        A.row_offsets = d_off;
        A.col_indices = (const int32_t*)d_col;
        A.values = d_val;
        rc = lw_spmv(schedule, &A, d_x, d_y, lanes, gs, tpb, d_ws, ws_b, stream);
    }
    if (!rc && y_b) rc = (int)cudaMemcpyAsync(y_host, d_y, y_b, cudaMemcpyDeviceToHost, s);
    cudaError_t fe = cudaFreeAsync(d, s);
    cudaError_t se = cudaStreamSynchronize(s);
    if (!rc) rc = (int)fe;
    if (!rc) rc = (int)se;
    return rc;
}

/* ---- SpMM ---------------------------------------------------------------------------- */

int lw_spmm_auto_lanes(int schedule, int64_t rows, int64_t nnz, int64_t n, int64_t gs, int64_t tpb,
                       int64_t* lanes_out) {
    if (!lanes_out || rows < 0 || nnz < 0 || n < 0) return LW_E_INVALID_ARG;
    if (schedule != LW_THREAD_MAPPED && schedule != LW_MERGE_PATH && schedule != LW_GROUP_MAPPED)
        return LW_E_INVALID_ARG;
    if (schedule == LW_GROUP_MAPPED && (gs < 1 || tpb < 1)) return LW_E_INVALID_ARG;
    *lanes_out = spmm_auto_lanes(schedule, rows, nnz, n, gs, tpb);
    return LW_OK;
}

size_t lw_spmm_workspace(int schedule, int64_t rows, int64_t nnz, int64_t n, int64_t lanes,
                         int32_t dtype) {
    (void)dtype;
    if (schedule != LW_MERGE_PATH || rows < 0 || nnz < 0 || n < 0 || lanes < 0) return 0;
    if (lanes == 0) lanes = spmm_auto_lanes(schedule, rows, nnz, n, 0, 0);
    return spmm_wo_workspace(lanes, n);
}

static int spmm_entry(int schedule, const lw_csr_t* A, const void* B, void* C, int64_t n,
                      int64_t lanes, int64_t gs, int64_t tpb, void* ws, size_t ws_bytes,
                      uintptr_t stream) {
    int rc = check_csr(A);
    if (rc) return rc;
    if (n < 0 || lanes < 0) return LW_E_INVALID_ARG;
    if (A->rows > 0 && n > 0 && !C) return LW_E_INVALID_ARG;
    if (A->nnz > 0 && n > 0 && !B) return LW_E_INVALID_ARG;
    if (schedule == LW_GROUP_MAPPED && (gs < 1 || tpb < 1)) return LW_E_INVALID_ARG;
    if (schedule != LW_THREAD_MAPPED && schedule != LW_MERGE_PATH && schedule != LW_GROUP_MAPPED)
        return LW_E_INVALID_ARG;
    if (lanes == 0) lanes = spmm_auto_lanes(schedule, A->rows, A->nnz, n, gs, tpb);
    return spmm(schedule, A, B, C, n, lanes, gs, tpb, ws, ws_bytes, (cudaStream_t)stream);
}

int lw_spmm_thread_mapped(const lw_csr_t* A, const void* B, void* C, int64_t n, int64_t lanes,
                          uintptr_t stream) {
    return spmm_entry(LW_THREAD_MAPPED, A, B, C, n, lanes, 0, 0, nullptr, 0, stream);
}

int lw_spmm_work_oriented(const lw_csr_t* A, const void* B, void* C, int64_t n, int64_t lanes,
                          void* ws, size_t ws_bytes, uintptr_t stream) {
    return spmm_entry(LW_MERGE_PATH, A, B, C, n, lanes, 0, 0, ws, ws_bytes, stream);
}

int lw_spmm_group_mapped(const lw_csr_t* A, const void* B, void* C, int64_t n, int64_t lanes,
                         int64_t gs, int64_t tpb, uintptr_t stream) {
    return spmm_entry(LW_GROUP_MAPPED, A, B, C, n, lanes, gs, tpb, nullptr, 0, stream);
}

int lw_spmm(int schedule, const lw_csr_t* A, const void* B, void* C, int64_t n, int64_t lanes,
            int64_t gs, int64_t tpb, void* ws, size_t ws_bytes, uintptr_t stream) {
    return spmm_entry(schedule, A, B, C, n, lanes, gs, tpb, ws, ws_bytes, stream);
}

/* ---- power-iteration normalisation ----------------------------------------------------- */

size_t lw_norm_workspace(int64_t n) { return n < 0 ? 0 : norm_workspace(n); }

int lw_vector_norm(const void* y, int64_t n, int32_t dtype, void* ws, size_t ws_bytes,
                   double* norm_out, uintptr_t stream) {
    if (n < 0 || (n > 0 && !y) || !norm_out || (dtype != LW_F32 && dtype != LW_F64))
        return LW_E_INVALID_ARG;
    if (!ws || ws_bytes < norm_workspace(n)) return LW_E_WORKSPACE;
    return vector_norm(y, n, dtype, ws, norm_out, (cudaStream_t)stream);
}

int lw_vector_scale(const void* y, int64_t n, int32_t dtype, const double* norm, void* x_out,
                    uintptr_t stream) {
    if (n < 0 || (n > 0 && (!y || !x_out)) || !norm || (dtype != LW_F32 && dtype != LW_F64))
        return LW_E_INVALID_ARG;
    return vector_scale(y, n, dtype, norm, x_out, (cudaStream_t)stream);
}

/* ---- SSSP / BFS ------------------------------------------------------------------------ */

size_t lw_frontier_workspace(int64_t n_vertices) {
    return n_vertices < 0 ? 0 : frontier_workspace(n_vertices);
}

static int check_graph(const lw_csr_t* G, int schedule, int64_t lanes, int64_t gs, int64_t tpb,
                       void* ws, size_t ws_bytes) {
    int rc = check_csr(G);
    if (rc) return rc;
    if (G->rows != G->cols || lanes < 0) return LW_E_INVALID_ARG;
    if (schedule != LW_THREAD_MAPPED && schedule != LW_MERGE_PATH && schedule != LW_GROUP_MAPPED)
        return LW_E_INVALID_ARG;
    if (schedule == LW_GROUP_MAPPED && (gs < 1 || tpb < 1)) return LW_E_INVALID_ARG;
    if (G->rows > 0x7fffffffLL) return LW_E_UNSUPPORTED;   // active lists are int32
    if (!ws || ws_bytes < frontier_workspace(G->rows)) return LW_E_WORKSPACE;
    return LW_OK;
}

int lw_frontier_compact(const uint8_t* mask, int64_t n, int32_t* active, int64_t* count_dev,
                        void* ws, size_t ws_bytes, uintptr_t stream) {
    if (n < 0 || (n > 0 && (!mask || !active)) || !count_dev) return LW_E_INVALID_ARG;
    if (!ws || ws_bytes < frontier_workspace(n)) return LW_E_WORKSPACE;
    return frontier_compact(mask, n, active, count_dev, ws, (cudaStream_t)stream);
}

int lw_sssp_pass(const lw_csr_t* G, const int32_t* active, int64_t n_active, double* dist,
                 uint8_t* out_frontier, int schedule, int64_t lanes, int64_t gs, int64_t tpb,
                 void* ws, size_t ws_bytes, uintptr_t stream) {
    int rc = check_graph(G, schedule, lanes, gs, tpb, ws, ws_bytes);
    if (rc) return rc;
    if (n_active < 0 || n_active > G->rows || (n_active > 0 && !active)) return LW_E_INVALID_ARG;
    if (G->rows > 0 && (!dist || !out_frontier)) return LW_E_INVALID_ARG;
    return sssp_pass(G, active, n_active, dist, out_frontier, schedule, lanes, gs, tpb, ws,
                     (cudaStream_t)stream);
}

int lw_bfs_pass(const lw_csr_t* G, const int32_t* active, int64_t n_active, int64_t* depth,
                int64_t next_depth, uint8_t* out_frontier, int schedule, int64_t lanes, int64_t gs,
                int64_t tpb, void* ws, size_t ws_bytes, uintptr_t stream) {
    int rc = check_graph(G, schedule, lanes, gs, tpb, ws, ws_bytes);
    if (rc) return rc;
    if (n_active < 0 || n_active > G->rows || (n_active > 0 && !active)) return LW_E_INVALID_ARG;
    if (G->rows > 0 && (!depth || !out_frontier)) return LW_E_INVALID_ARG;
    return bfs_pass(G, active, n_active, depth, next_depth, out_frontier, schedule, lanes, gs, tpb,
                    ws, (cudaStream_t)stream);
}

int lw_sssp(const lw_csr_t* G, int64_t source, double* dist, int schedule, int64_t lanes,
            int64_t gs, int64_t tpb, void* ws, size_t ws_bytes, int64_t* passes_out,
            uintptr_t stream) {
    int rc = check_graph(G, schedule, lanes, gs, tpb, ws, ws_bytes);
    if (rc) return rc;
    if (source < 0 || source >= G->rows || !dist) return LW_E_INVALID_ARG;
    return sssp_run(G, source, dist, schedule, lanes, gs, tpb, ws, passes_out, (cudaStream_t)stream);
}

int lw_bfs(const lw_csr_t* G, int64_t source, int64_t* depth, int schedule, int64_t lanes,
           int64_t gs, int64_t tpb, void* ws, size_t ws_bytes, int64_t* passes_out,
           uintptr_t stream) {
    int rc = check_graph(G, schedule, lanes, gs, tpb, ws, ws_bytes);
    if (rc) return rc;
    if (source < 0 || source >= G->rows || !depth) return LW_E_INVALID_ARG;
    return bfs_run(G, source, depth, schedule, lanes, gs, tpb, ws, passes_out, (cudaStream_t)stream);
}

int lw_rmat_keys(int32_t scale, int64_t edge_begin, int64_t n_edges, uint32_t t_a, uint32_t t_ab,
                 uint32_t t_abc, uint64_t seed, int64_t* keys, uintptr_t stream) {
    return rmat_keys(scale, edge_begin, n_edges, t_a, t_ab, t_abc, seed, keys, (cudaStream_t)stream);
}

int lw_uniform_keys(int64_t space, int64_t begin, int64_t n, uint64_t seed, int64_t* keys,
                    uintptr_t stream) {
    return uniform_keys(space, begin, n, seed, keys, (cudaStream_t)stream);
}

int lw_hash_values(const int64_t* keys, int64_t n, uint64_t seed, int32_t dtype, void* values,
                   uintptr_t stream) {
    return hash_values(keys, n, seed, dtype, values, (cudaStream_t)stream);
}

}  // extern "C"
