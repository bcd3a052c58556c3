// hotx.cu — hot-x column packing: a one-time inspector over a CSR's column
// indices for the work_oriented SpMV (lw_spmv_work_oriented_hotx).
//
// Why: on power-law matrices (C3) the SpMV is bound by the SM's
// L1->L2 request rate, one request per x gather that misses L1. The most
// gathered columns are scattered over x, so each pins a whole 32-byte L1 sector
// for one useful value and the cold gathers evict them. The inspector relabels
// the (at most max_hot) most gathered columns to dense slots of a packed copy
// xh (8 fp32 values per sector) that the SpMV keeps in L1, and marks them with
// bit 31 of the column index:
//     col_packed[a] = slot(col[a]) | 0x80000000   if col[a] is hot
//                   = col[a]                        otherwise.
// The products, their order and every sum are unchanged, so y is bit-identical
// to lw_spmv_work_oriented's.
//
// Hot set: H = { c : count(c) >= T } with count(c) the number of atoms in
// column c and T the smallest threshold >= 2 with |H| <= max_hot (a column
// gathered once gains nothing). T is found exactly by a two-pass radix select
// over the 32-bit counts (high 16 bits, then low 16 bits of the boundary bin);
// the two 64 K-bin histograms are read by the host between passes. Slots are in
// ascending column order (one CTA sorts the collected set), so col_packed and
// hot_cols are deterministic.
#include <climits>
#include <mutex>

#include "lw_common.cuh"

namespace lw {

int sm_count();

constexpr int HX_BINS = 1 << 16;
constexpr int HX_MAX_HOT = 32768;   // sorted in one CTA's shared memory (128 KB)

__global__ void k_hx_count(const int32_t* __restrict__ col, int64_t nnz, int32_t* __restrict__ counts) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
         i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(counts + col[i], 1);
}

// pass 0: bin = count >> 16 over every column; pass 1: bin = count & 0xffff over
// the columns whose high half equals hi. Lanes with equal bins add once per warp;
// the low bins (where nearly every column of a power-law matrix falls: bin 0 in
// pass 0, small counts in pass 1) go to a per-CTA shared histogram flushed once,
// instead of every warp's atomic hitting the same few global words (pass 0 + 1:
// 1.15 -> ~0.1 ms on C3).
constexpr int HX_SBINS = 1024;
__global__ void __launch_bounds__(256) k_hx_hist(const int32_t* __restrict__ counts, int64_t cols, int pass,
                                                 uint32_t hi, uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_h[HX_SBINS];
    for (int i = threadIdx.x; i < HX_SBINS; i += blockDim.x) s_h[i] = 0u;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < cols; base += stride) {
        const int64_t c = base + threadIdx.x;
        int bin = -1;
        if (c < cols) {
            const uint32_t v = (uint32_t)counts[c];
            if (pass == 0) bin = (int)(v >> 16);
            else if ((v >> 16) == hi) bin = (int)(v & 0xffffu);
        }
        const unsigned act = __ballot_sync(0xffffffffu, bin >= 0);
        if (bin >= 0) {
            const unsigned peers = __match_any_sync(act, bin);
            if ((threadIdx.x & 31) == __ffs(peers) - 1) {
                if (bin < HX_SBINS) atomicAdd(s_h + bin, (uint32_t)__popc(peers));
                else atomicAdd(hist + bin, (uint32_t)__popc(peers));
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < HX_SBINS; i += blockDim.x)
        if (s_h[i]) atomicAdd(hist + i, s_h[i]);
}

__global__ void k_hx_collect(const int32_t* __restrict__ counts, int64_t cols, uint32_t thr,
                             int32_t* __restrict__ hot, int32_t* __restrict__ n_hot) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
         c += (int64_t)gridDim.x * blockDim.x)
        if ((uint32_t)counts[c] >= thr) hot[atomicAdd(n_hot, 1)] = (int32_t)c;
}

// one CTA: bitonic sort of the n collected columns (padded with INT_MAX to a power of two)
__global__ void __launch_bounds__(1024) k_hx_sort(int32_t* __restrict__ hot, int n, int n2) {
    extern __shared__ int32_t sh[];
    for (int i = threadIdx.x; i < n2; i += blockDim.x) sh[i] = i < n ? hot[i] : INT_MAX;
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const bool up = (i & k) == 0;
                    const int32_t a = sh[i], b = sh[p];
                    if ((a > b) == up) { sh[i] = b; sh[p] = a; }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < n; i += blockDim.x) hot[i] = sh[i];
}

__global__ void k_hx_slots(const int32_t* __restrict__ hot, int n, int32_t* __restrict__ slot_of) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) slot_of[hot[i]] = i;
}

__global__ void k_hx_remap(const int32_t* __restrict__ col, int64_t nnz,
                           const int32_t* __restrict__ slot_of, int32_t* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = col[i], s = slot_of[c];
        out[i] = s >= 0 ? (int32_t)((uint32_t)s | 0x80000000u) : c;
    }
}

// ---- symmetric permutation P A P^T (degree relabeling for the iterated SpMV) ----
// Row i' of the result is row order[i'] of A with every column c renamed
// rank[c] (rank = order^-1); a row's atoms keep their order, so each row sum
// adds the same products in the same sequence. One warp per output row, lanes
// striding the row (coalesced on both sides); rows of any length.
template <class OffT, class ValT>
__global__ void k_csr_permute(const OffT* __restrict__ off, const int32_t* __restrict__ col,
                              const ValT* __restrict__ val, const int64_t* __restrict__ order,
                              const int32_t* __restrict__ rank, const OffT* __restrict__ off_out,
                              int64_t rows, int32_t* __restrict__ col_out, ValT* __restrict__ val_out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
        const int64_t src = order[r];
        const int64_t a0 = (int64_t)off[src], len = (int64_t)off[src + 1] - a0, b0 = (int64_t)off_out[r];
        for (int64_t k = lane; k < len; k += 32) {
            col_out[b0 + k] = rank[col[a0 + k]];
            val_out[b0 + k] = val[a0 + k];
        }
    }
}

int csr_permute(const lw_csr_t* A, const int64_t* order, const int32_t* rank, const void* off_out,
                int32_t* col_out, void* val_out, cudaStream_t s) {
    if (!A || A->rows != A->cols || (A->rows > 0 && (!order || !rank || !off_out)) ||
        (A->nnz > 0 && (!col_out || !val_out)))
        return LW_E_INVALID_ARG;
    if (A->rows == 0) return LW_OK;
    const unsigned grid = (unsigned)sm_count() * 8;
    if (A->offset_bits == 32) {
        if (A->dtype == LW_F32)
            k_csr_permute<int32_t, float><<<grid, 256, 0, s>>>((const int32_t*)A->row_offsets, A->col_indices,
                (const float*)A->values, order, rank, (const int32_t*)off_out, A->rows, col_out, (float*)val_out);
        else
            k_csr_permute<int32_t, double><<<grid, 256, 0, s>>>((const int32_t*)A->row_offsets, A->col_indices,
                (const double*)A->values, order, rank, (const int32_t*)off_out, A->rows, col_out, (double*)val_out);
    } else {
        if (A->dtype == LW_F32)
            k_csr_permute<int64_t, float><<<grid, 256, 0, s>>>((const int64_t*)A->row_offsets, A->col_indices,
                (const float*)A->values, order, rank, (const int64_t*)off_out, A->rows, col_out, (float*)val_out);
        else
            k_csr_permute<int64_t, double><<<grid, 256, 0, s>>>((const int64_t*)A->row_offsets, A->col_indices,
                (const double*)A->values, order, rank, (const int64_t*)off_out, A->rows, col_out, (double*)val_out);
    }
    LW_LAUNCH_CHECK();
    return LW_OK;
}

static size_t hx_align(size_t v) { return (v + 255) / 256 * 256; }

size_t hotx_build_workspace(int64_t cols) {
    return hx_align((size_t)cols * 4) + hx_align((size_t)HX_BINS * 4) + 256;
}

int hotx_build(const lw_csr_t* A, int32_t max_hot, int32_t* col_packed, int32_t* hot_cols,
               int32_t* n_hot_out, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (!n_hot_out || max_hot < 0 || max_hot > HX_MAX_HOT || (A->nnz > 0 && !col_packed) ||
        (max_hot > 0 && !hot_cols) || A->cols >= ((int64_t)1 << 31))
        return LW_E_INVALID_ARG;
    *n_hot_out = 0;
    if (A->nnz == 0) return LW_OK;
    if (!ws || ws_bytes < hotx_build_workspace(A->cols)) return LW_E_WORKSPACE;
    unsigned char* w = (unsigned char*)ws;
    int32_t* counts = (int32_t*)w;                                  // later: slot_of
    uint32_t* hist = (uint32_t*)(w + hx_align((size_t)A->cols * 4));
    int32_t* n_dev = (int32_t*)(w + hx_align((size_t)A->cols * 4) + hx_align((size_t)HX_BINS * 4));
    const unsigned grid = (unsigned)sm_count() * 8;

    uint32_t thr = UINT_MAX;   // no hot set unless a threshold >= 2 fits
    if (max_hot > 0) {
        LW_TRY(cudaMemsetAsync(counts, 0, (size_t)A->cols * 4, s));
        k_hx_count<<<grid, 256, 0, s>>>(A->col_indices, A->nnz, counts);
        LW_LAUNCH_CHECK();
        // radix select: smallest thr >= 2 with |{count >= thr}| <= max_hot
        static uint32_t h[HX_BINS];   // host copies of the histograms (guarded below)
        static std::mutex* mu = new std::mutex;
        std::lock_guard<std::mutex> lk(*mu);
        LW_TRY(cudaMemsetAsync(hist, 0, (size_t)HX_BINS * 4, s));
        k_hx_hist<<<grid, 256, 0, s>>>(counts, A->cols, 0, 0u, hist);
        LW_LAUNCH_CHECK();
        LW_TRY(cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, s));
        LW_TRY(cudaStreamSynchronize(s));
        uint64_t above = 0;   // columns in bins > b
        int b = HX_BINS - 1;
        for (; b >= 0; --b) {
            if (above + h[b] > (uint64_t)max_hot) break;
            above += h[b];
        }
        if (b < 0) {
            thr = 2;   // every column fits
        } else {
            // refine inside bin b: columns with count>>16 == b, by their low half
            LW_TRY(cudaMemsetAsync(hist, 0, (size_t)HX_BINS * 4, s));
            k_hx_hist<<<grid, 256, 0, s>>>(counts, A->cols, 1, (uint32_t)b, hist);
            LW_LAUNCH_CHECK();
            LW_TRY(cudaMemcpyAsync(h, hist, sizeof(h), cudaMemcpyDeviceToHost, s));
            LW_TRY(cudaStreamSynchronize(s));
            int l = HX_BINS - 1;
            for (; l >= 0; --l) {
                if (above + h[l] > (uint64_t)max_hot) break;
                above += h[l];
            }
            thr = ((uint32_t)b << 16) + (uint32_t)(l + 1);   // l + 1 may carry into b + 1
        }
        if (thr < 2) thr = 2;
    }
    int32_t n = 0;
    if (thr != UINT_MAX) {
        LW_TRY(cudaMemsetAsync(n_dev, 0, 4, s));
        k_hx_collect<<<grid, 256, 0, s>>>(counts, A->cols, thr, hot_cols, n_dev);
        LW_LAUNCH_CHECK();
        LW_TRY(cudaMemcpyAsync(&n, n_dev, 4, cudaMemcpyDeviceToHost, s));
        LW_TRY(cudaStreamSynchronize(s));
        if (n > max_hot) return LW_E_UNSUPPORTED;   // cannot happen: thr bounds the set
    }
    if (n > 0) {
        int n2 = 1;
        while (n2 < n) n2 <<= 1;
        const size_t sh = (size_t)n2 * 4;
        LW_TRY(cudaFuncSetAttribute(k_hx_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        k_hx_sort<<<1, 1024, sh, s>>>(hot_cols, n, n2);
        LW_LAUNCH_CHECK();
    }
    LW_TRY(cudaMemsetAsync(counts, 0xff, (size_t)A->cols * 4, s));   // slot_of = -1
    if (n > 0) {
        k_hx_slots<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(hot_cols, n, counts);
        LW_LAUNCH_CHECK();
    }
    k_hx_remap<<<grid, 256, 0, s>>>(A->col_indices, A->nnz, counts, col_packed);
    LW_LAUNCH_CHECK();
    *n_hot_out = n;
    return LW_OK;
}

}  // namespace lw
