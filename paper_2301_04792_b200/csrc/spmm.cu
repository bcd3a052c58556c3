// spmm.cu — C = A B (B dense row-major [cols x n], C row-major [rows x n]) under
// the three schedules. The paper's SpMM is "a loop over the columns of B wrapped
// around the SpMV body" (Listing 4); the reference restates it as
// kernels.spmm (kernels.py:129-175) over _fast.spmm_{thread_mapped,merge_path,
// group_mapped} (_fast.py:80-144). The schedules -- which lane owns which tiles
// and atoms -- are exactly the SpMV ones; only the per-atom work widens from one
// x value to one row of B.
//
// Device mapping: a lane is a TEAM of TS threads (TS = power of two <= 32) that
// covers a slab of TS*VEC consecutive columns, VEC columns per thread with one
// 16-byte load of B / store of C (VEC = 4 fp32, 2 fp64; 1 when n or the pointers
// do not allow it). Slabs wider than 32*VEC are walked one after the other, re-reading the
// lane's atoms (the reference's column loop). A team reads each atom's column
// index and value once (the same address for the whole team, one L1 request)
// and gathers a contiguous TS*VEC-wide row segment of B. Sums are fp64 and follow
// the atom order of the reference loops, so integer data is bit-exact.
#include <algorithm>

#include "lw_common.cuh"

namespace lw {

int mp_bound_tiles(const lw_csr_t* A, int64_t lanes, int64_t J, int64_t S, int64_t* tiles,
                   cudaStream_t s);
int64_t group_auto_lanes(int64_t rows, int64_t gs, int64_t tpb);

constexpr int MM_NT = 256;   // threads per CTA (a multiple of every team size)
constexpr int MM_U = 8;      // atoms per batch: col/val/B loads in flight per thread

// VEC consecutive values of B / C (16-byte vectors: float4 / double2)
template <class ValT, int VEC>
__device__ __forceinline__ void ld_row(const ValT* p, ValT* v) {
    if constexpr (VEC == 4) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else if constexpr (VEC == 2) {
        const double2 q = __ldg(reinterpret_cast<const double2*>(p));
        v[0] = q.x; v[1] = q.y;
    } else {
        v[0] = __ldg(p);
    }
}
template <class ValT, int VEC, class AccT = double>
__device__ __forceinline__ void st_row(ValT* p, const AccT* a) {
    if constexpr (VEC == 4) {
        *reinterpret_cast<float4*>(p) = make_float4((float)a[0], (float)a[1], (float)a[2], (float)a[3]);
    } else if constexpr (VEC == 2) {
        *reinterpret_cast<double2*>(p) = make_double2((double)a[0], (double)a[1]);
    } else {
        p[0] = (ValT)a[0];
    }
}

// atoms per batch of the atom-major walk: about 16 B-row values per thread in flight
// (16-byte vectors: 4 atoms; fp64 with 8 atoms spilled and was 25-33% slower)
// (6 or 8 atoms with fp32 vectors spilled: 31-39% slower)
template <int VEC>
struct MmU {
    static constexpr int U = VEC >= 2 ? 4 : 8;
};

// Accumulate atoms [a, a+cnt) (cnt <= MM_U, all in the same row) into acc.
template <class OffT, class ValT, int VEC>
__device__ __forceinline__ void mm_batch(const Csr<OffT, ValT>& A, const ValT* __restrict__ B,
                                         int64_t n, int64_t c, bool active, int64_t a, int cnt,
                                         double* acc) {
    int32_t col[MM_U];
    ValT val[MM_U];
#pragma unroll
    for (int k = 0; k < MM_U; ++k) {
        col[k] = k < cnt ? __ldg(A.col + a + k) : 0;
        val[k] = k < cnt ? __ldg(A.val + a + k) : (ValT)0;
    }
    ValT b[MM_U][VEC];
#pragma unroll
    for (int k = 0; k < MM_U; ++k) {
        if (active && k < cnt) ld_row<ValT, VEC>(B + (int64_t)col[k] * n + c, b[k]);
        else
#pragma unroll
            for (int j = 0; j < VEC; ++j) b[k][j] = (ValT)0;
    }
    if constexpr (sizeof(ValT) == 4) {
        // fp32: the batch is summed in fp32 and folded into the fp64 sum once
        // (an fp64 FMA per product was 28-34% slower on C2u)
        ValT part[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) part[j] = (ValT)0;
#pragma unroll
        for (int k = 0; k < MM_U; ++k)
#pragma unroll
            for (int j = 0; j < VEC; ++j) part[j] = fma(val[k], b[k][j], part[j]);
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] += (double)part[j];
    } else {
#pragma unroll
        for (int k = 0; k < MM_U; ++k)
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc[j] = fma((double)val[k], (double)b[k][j], acc[j]);
    }
}

// Full sum of atoms [s, e) for one slab (sequential in atom order).
template <class OffT, class ValT, int VEC>
__device__ __forceinline__ void mm_range(const Csr<OffT, ValT>& A, const ValT* __restrict__ B,
                                         int64_t n, int64_t c, bool active, int64_t s, int64_t e,
                                         double* acc) {
    for (int64_t a = s; a < e; a += MM_U) {
        const int cnt = (int)min((int64_t)MM_U, e - a);
        mm_batch<OffT, ValT, VEC>(A, B, n, c, active, a, cnt, acc);
    }
}

// ---- thread_mapped: lane l owns tiles l, l+P, ... (_fast.py:80-90) --------------------
// Resident MM_NT-thread CTAs the thread-mapped kernel's registers must allow: 4 ->
// 64 registers (80 uncapped for fp32 vectors): fp32 n = 4 / 16 / 64, C3 78 / 117 /
// 181 -> 61 / 87 / 131 ms, C2u n = 16 / 64 -17 / -19%, C2b n = 16 -12%, n = 4 +-3%.
// (5 -> 48 registers spills 104 B.)
#ifndef LW_MM_TM_MINB
#define LW_MM_TM_MINB 4
#endif
template <class OffT, class ValT, int VEC>
__global__ void __launch_bounds__(MM_NT, LW_MM_TM_MINB)
    k_spmm_thread_mapped(Csr<OffT, ValT> A, const ValT* __restrict__ B, ValT* __restrict__ C,
                         int64_t n, int64_t lanes, int lg_ts) {
    const int64_t gt = (int64_t)blockIdx.x * MM_NT + threadIdx.x;
    const int64_t lane = gt >> lg_ts;
    const int tl = (int)(gt & ((1 << lg_ts) - 1));
    if (lane >= lanes) return;
    const int64_t sw = ((int64_t)VEC) << lg_ts;   // slab width
    for (int64_t t = lane; t < A.rows; t += lanes) {
        const int64_t s = (int64_t)__ldg(A.off + t), e = (int64_t)__ldg(A.off + t + 1);
        for (int64_t cs = 0; cs < n; cs += sw) {
            const int64_t c = cs + (int64_t)tl * VEC;
            const bool active = c < n;
            double acc[VEC];
#pragma unroll
            for (int j = 0; j < VEC; ++j) acc[j] = 0.0;
            mm_range<OffT, ValT, VEC>(A, B, n, c, active, s, e, acc);
            if (active) st_row<ValT, VEC>(C + t * n + c, acc);
        }
    }
}

// ---- work_oriented (merge path): even share of rows+nnz per lane (_fast.py:93-118) ----
// Lane k walks diagonals [min(k*items,total), min((k+1)*items,total)): rows
// [t0, t1) end inside its slice and are assigned; the partial row t1 becomes the
// lane's carry (n values), added in lane order by k_spmm_carry_fixup.
#ifndef LW_MM_WO_MINB
#define LW_MM_WO_MINB 4
#endif
template <class OffT, class ValT, int VEC>
__global__ void __launch_bounds__(MM_NT, LW_MM_WO_MINB)
    k_spmm_work_oriented(Csr<OffT, ValT> A, const ValT* __restrict__ B, ValT* __restrict__ C,
                         int64_t n, int64_t lanes, int64_t items, int lg_ts,
                         const int64_t* __restrict__ bound_tile, int64_t* __restrict__ carry_tile,
                         double* __restrict__ carry_val) {
    constexpr int U = MmU<VEC>::U;
    const int64_t gt = (int64_t)blockIdx.x * MM_NT + threadIdx.x;
    const int64_t lane = gt >> lg_ts;
    const int tl = (int)(gt & ((1 << lg_ts) - 1));
    if (lane >= lanes) return;
    const int64_t total = A.rows + A.nnz;
    const int64_t d0 = min(lane * items, total), d1 = min((lane + 1) * items, total);
    const int64_t t0 = bound_tile[lane], t1 = bound_tile[lane + 1];
    const int64_t a0 = d0 - t0, a1 = d1 - t1;
    const int64_t sw = ((int64_t)VEC) << lg_ts;
    // the partial row t1 covers atoms [ts, a1)
    const int64_t ts = t1 > t0 ? (int64_t)__ldg(A.off + t1) : a0;
    const bool carry = a1 > ts;
    if (tl == 0) carry_tile[lane] = carry ? t1 : -1;
    for (int64_t cs = 0; cs < n; cs += sw) {
        const int64_t c = cs + (int64_t)tl * VEC;
        const bool active = c < n;
        // atom-major walk: batches of U atoms cross row ends, so every batch
        // keeps U gathers of B in flight however short the rows are; the next
        // row end is loaded one row ahead
        int64_t t = t0;
        int64_t re = t < t1 ? (int64_t)__ldg(A.off + t + 1) : a1;
        int64_t re2 = t + 1 < t1 ? (int64_t)__ldg(A.off + t + 2) : a1;
        // fp32: products are summed in fp32 within a batch of U atoms and folded
        // into the fp64 row sum once per batch (4 fp32 FMAs per fp64 add: -23%
        // time on C3 n=16 against fp64 FMAs for every product); fp64 sums directly
        constexpr bool kBatchPart = sizeof(ValT) == 4;
        double acc[VEC];
        ValT part[VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) { acc[v] = 0.0; part[v] = (ValT)0; }
        auto finish_row = [&]() {
            if constexpr (kBatchPart) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) { acc[v] += (double)part[v]; part[v] = (ValT)0; }
            }
            if (active) st_row<ValT, VEC>(C + t * n + c, acc);
#pragma unroll
            for (int v = 0; v < VEC; ++v) acc[v] = 0.0;
            ++t;
            re = re2;
            re2 = t + 1 < t1 ? (int64_t)__ldg(A.off + t + 2) : a1;
        };
        for (int64_t a = a0; a < a1; a += U) {
            const int cnt = (int)min((int64_t)U, a1 - a);
            int32_t col[U];
            ValT val[U];
            ValT b[U][VEC];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                col[k] = k < cnt ? __ldg(A.col + a + k) : 0;
                val[k] = k < cnt ? __ldg(A.val + a + k) : (ValT)0;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if (active && k < cnt) ld_row<ValT, VEC>(B + (int64_t)col[k] * n + c, b[k]);
                else
#pragma unroll
                    for (int v = 0; v < VEC; ++v) b[k][v] = (ValT)0;
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if (k < cnt) {
                    while (t < t1 && re <= a + k) finish_row();
                    if constexpr (kBatchPart) {
#pragma unroll
                        for (int v = 0; v < VEC; ++v) part[v] = fma(val[k], b[k][v], part[v]);
                    } else {
#pragma unroll
                        for (int v = 0; v < VEC; ++v) acc[v] = fma((double)val[k], (double)b[k][v], acc[v]);
                    }
                }
            }
            if constexpr (kBatchPart) {
#pragma unroll
                for (int v = 0; v < VEC; ++v) { acc[v] += (double)part[v]; part[v] = (ValT)0; }
            }
        }
        while (t < t1) finish_row();   // rows ending at a1, and empty rows
        if (carry && active)
#pragma unroll
            for (int v = 0; v < VEC; ++v) carry_val[lane * n + c + v] = acc[v];
    }
}

// Ordered carry fix-up, one thread per (carry, column): the head of every run of
// carries into one row sums the run in lane order and adds it (kernels.py:160-162).
template <class ValT>
__global__ void k_spmm_carry_fixup(const int64_t* __restrict__ carry_tile,
                                   const double* __restrict__ carry_val, int64_t lanes, int64_t n,
                                   ValT* __restrict__ C) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= lanes * n) return;
    const int64_t k = i / n, c = i - k * n;
    const int64_t r = carry_tile[k];
    if (r < 0) return;
    for (int64_t m = k - 1; m >= 0; --m) {
        const int64_t t = carry_tile[m];
        if (t == r) return;   // not the head of its run
        if (t >= 0) break;
    }
    double s = 0.0;
    for (int64_t m = k; m < lanes; ++m) {
        const int64_t t = carry_tile[m];
        if (t < 0) continue;
        if (t != r) break;
        s += carry_val[m * n + c];
    }
    C[r * n + c] = (ValT)((double)C[r * n + c] + s);
}

// ---- group_mapped: groups own blocks of tiles, members stride atoms (_fast.py:121-144) --
// The reference adds v * B[src, c] into C[tile, c] member by member: member 0's
// atoms of the tile in increasing order, then member 1's, ... (member m of the
// group owning the tile's block takes block-local atoms m, m + M, ...). One team
// per tile replays that order per column with unfused fp64 multiply and add
// (the SpMV k_group_tiles walk): C is written once per tile, run-to-run
// identical and, for fp64 data, bit-identical to the reference — no atomics,
// no zeroing pass.
constexpr int GT_U = 4;   // atoms per residue batch (loads in flight)
// Resident MM_NT-thread CTAs the group-tile kernel's registers must allow: 4 ->
// 64 registers (73 uncapped), fp32 n = 4 / 16 / 64: C2u 0.286 / 0.719 / 2.71 ->
// 0.275 / 0.600 / 2.18 ms, C2b 0.245 / 0.497 / 1.96 -> 0.249 / 0.431 / 1.66, C3
// -1..-3%. (5 -> 48 registers spills 60-92 B.)
#ifndef LW_MM_GT_MINB
#define LW_MM_GT_MINB 4
#endif
template <class OffT, class ValT, int VEC>
__global__ void __launch_bounds__(MM_NT, LW_MM_GT_MINB)
    k_spmm_group_tiles(Csr<OffT, ValT> A, const ValT* __restrict__ B, ValT* __restrict__ C, int64_t n,
                       int64_t lanes, int64_t gs, int64_t tpb, int lg_ts) {
    const int64_t gt = (int64_t)blockIdx.x * MM_NT + threadIdx.x;
    const int64_t t = gt >> lg_ts;
    const int tl = (int)(gt & ((1 << lg_ts) - 1));
    if (t >= A.rows) return;
    const int64_t groups = (lanes + gs - 1) / gs;
    const int64_t b = t / tpb, g = b % groups;
    const int64_t M = min(gs, lanes - g * gs);
    const int64_t base = (int64_t)__ldg(A.off + b * tpb);
    const int64_t e0 = (int64_t)__ldg(A.off + t) - base, e1 = (int64_t)__ldg(A.off + t + 1) - base;
    const int64_t sw = ((int64_t)VEC) << lg_ts;   // slab width
    for (int64_t cs = 0; cs < n; cs += sw) {
        const int64_t c = cs + (int64_t)tl * VEC;
        if (c >= n) continue;
        double acc[VEC];
#pragma unroll
        for (int j = 0; j < VEC; ++j) acc[j] = 0.0;
        if (e1 - e0 >= GT_U * M) {
            // long tile: member by member (same order), GT_U of a member's atoms
            // (stride M) in flight per batch — no walker arithmetic per atom
            const int64_t r0 = e0 % M;
            auto member = [&](int64_t i) {
                for (int64_t k0 = e0 + i; k0 < e1; k0 += GT_U * M) {
                    int32_t col[GT_U];
                    double v[GT_U];
#pragma unroll
                    for (int u = 0; u < GT_U; ++u) {
                        const int64_t k = k0 + u * M < e1 ? k0 + u * M : k0;
                        col[u] = __ldg(A.col + base + k);
                        v[u] = (double)__ldg(A.val + base + k);
                    }
                    ValT bv[GT_U][VEC];
#pragma unroll
                    for (int u = 0; u < GT_U; ++u) ld_row<ValT, VEC>(B + (int64_t)col[u] * n + c, bv[u]);
#pragma unroll
                    for (int u = 0; u < GT_U; ++u)
                        if (k0 + u * M < e1)
#pragma unroll
                            for (int j = 0; j < VEC; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(v[u], (double)bv[u][j]));
                }
            };
            for (int64_t i = M - r0; i < M; ++i) member(i);   // wrapped residues 0, 1, ... first
            for (int64_t i = 0; i < M - r0; ++i) member(i);
            st_row<ValT, VEC>(C + t * n + c, acc);
            continue;
        }
        MemberMajorWalk w(e0, e1, M);
        for (int64_t p0 = w.next(); p0 >= 0;) {   // GT_U atoms' loads in flight, then the ordered adds
            int64_t k[GT_U];
            k[0] = p0;
#pragma unroll
            for (int u = 1; u < GT_U; ++u) k[u] = k[u - 1] >= 0 ? w.next() : -1;
            int32_t col[GT_U];
            double v[GT_U];
#pragma unroll
            for (int u = 0; u < GT_U; ++u) {
                col[u] = k[u] >= 0 ? __ldg(A.col + base + k[u]) : 0;
                v[u] = k[u] >= 0 ? (double)__ldg(A.val + base + k[u]) : 0.0;
            }
            ValT bv[GT_U][VEC];
#pragma unroll
            for (int u = 0; u < GT_U; ++u) {
                if (k[u] >= 0) ld_row<ValT, VEC>(B + (int64_t)col[u] * n + c, bv[u]);
                else
#pragma unroll
                    for (int j = 0; j < VEC; ++j) bv[u][j] = (ValT)0;
            }
#pragma unroll
            for (int u = 0; u < GT_U; ++u)
                if (k[u] >= 0)
#pragma unroll
                    for (int j = 0; j < VEC; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(v[u], (double)bv[u][j]));
            p0 = k[GT_U - 1] >= 0 ? w.next() : -1;
        }
        st_row<ValT, VEC>(C + t * n + c, acc);
    }
}

// ---- host side ------------------------------------------------------------------------
struct MmShape {
    int vec, lg_ts;
};

template <class ValT>
static MmShape mm_shape(int64_t n, const void* B, const void* C) {
    constexpr int V = 16 / (int)sizeof(ValT);
    const bool vec = n % V == 0 && ((uintptr_t)B % 16 == 0) && ((uintptr_t)C % 16 == 0);
    const int vw = vec ? V : 1;
    const int64_t need = (n + vw - 1) / vw;   // threads to cover n columns
    int lg = 0;
    while ((1 << lg) < need && lg < 5) ++lg;
    return MmShape{vw, lg};
}

static unsigned mm_grid(int64_t lanes, int lg_ts) {
    return (unsigned)ceil_div((lanes << lg_ts), MM_NT);
}

int64_t mm_wo_items_target() { return 256; }

int64_t spmm_auto_lanes(int schedule, int64_t rows, int64_t nnz, int64_t n, int64_t gs,
                        int64_t tpb) {
    int lg = 0;
    const int64_t need = n > 0 ? (n + 3) / 4 : 1;
    while ((1 << lg) < need && lg < 5) ++lg;
    switch (schedule) {
        case LW_THREAD_MAPPED: {
            const int64_t cap = ((int64_t)sm_count() * 2048) >> lg;
            const int64_t p = ceil_div(rows > 0 ? rows : 1, 64) * 64;
            return p < cap ? p : cap;
        }
        case LW_MERGE_PATH: {
            // 256 items per lane on large inputs; smaller inputs get shorter lanes
            // (down to 16 items) so that ~256 teams per SM still have work
            const int64_t total = rows + nnz;
            if (total <= 0) return 1;
            const int64_t teams = ((int64_t)sm_count() * 2048) >> lg;
            const int64_t items = std::max<int64_t>(16, std::min<int64_t>(mm_wo_items_target(),
                                                                          ceil_div(total, teams)));
            return ceil_div(total, items);
        }
        default: return group_auto_lanes(rows, gs, tpb);
    }
}

size_t spmm_wo_workspace(int64_t lanes, int64_t n) {
    auto up = [](size_t b) { return (b + 255) / 256 * 256; };
    return up((size_t)(lanes + 1) * 8) + up((size_t)lanes * 8) + up((size_t)lanes * (size_t)n * 8);
}

template <class OffT, class ValT>
static int spmm_typed(int schedule, const lw_csr_t* H, const void* Bp, void* Cp, int64_t n,
                      int64_t lanes, int64_t gs, int64_t tpb, void* ws, cudaStream_t s) {
    Csr<OffT, ValT> A{H->rows, H->cols, H->nnz, (const OffT*)H->row_offsets, H->col_indices,
                      (const ValT*)H->values};
    const ValT* B = (const ValT*)Bp;
    ValT* C = (ValT*)Cp;
    const MmShape sh = mm_shape<ValT>(n, Bp, Cp);
    const unsigned grid = mm_grid(lanes, sh.lg_ts);
    constexpr int V = 16 / (int)sizeof(ValT);
#define LW_MM_DISPATCH(KERN, ...)                                                      \
    do {                                                                               \
        if (sh.vec == V) KERN<OffT, ValT, V><<<grid, MM_NT, 0, s>>>(__VA_ARGS__);      \
        else KERN<OffT, ValT, 1><<<grid, MM_NT, 0, s>>>(__VA_ARGS__);                  \
    } while (0)
    switch (schedule) {
        case LW_THREAD_MAPPED:
            LW_MM_DISPATCH(k_spmm_thread_mapped, A, B, C, n, lanes, sh.lg_ts);
            LW_LAUNCH_CHECK();
            return LW_OK;
        case LW_MERGE_PATH: {
            auto up = [](size_t b) { return (b + 255) / 256 * 256; };
            unsigned char* w = (unsigned char*)ws;
            int64_t* tiles = (int64_t*)w;
            int64_t* c_tile = (int64_t*)(w + up((size_t)(lanes + 1) * 8));
            double* c_val = (double*)(w + up((size_t)(lanes + 1) * 8) + up((size_t)lanes * 8));
            const int64_t total = A.rows + A.nnz;
            const int64_t items = total > 0 ? ceil_div(total, lanes) : 0;
            int rc = mp_bound_tiles(H, lanes, 1, items, tiles, s);
            if (rc) return rc;
            LW_MM_DISPATCH(k_spmm_work_oriented, A, B, C, n, lanes, items, sh.lg_ts, tiles, c_tile,
                           c_val);
            LW_LAUNCH_CHECK();
            const int64_t work = lanes * n;
            k_spmm_carry_fixup<ValT><<<(unsigned)ceil_div(work, 256), 256, 0, s>>>(c_tile, c_val,
                                                                                  lanes, n, C);
            LW_LAUNCH_CHECK();
            return LW_OK;
        }
        case LW_GROUP_MAPPED: {
            const unsigned tgrid = mm_grid(A.rows, sh.lg_ts);   // one team per tile
            if (sh.vec == V) k_spmm_group_tiles<OffT, ValT, V><<<tgrid, MM_NT, 0, s>>>(A, B, C, n, lanes, gs, tpb, sh.lg_ts);
            else k_spmm_group_tiles<OffT, ValT, 1><<<tgrid, MM_NT, 0, s>>>(A, B, C, n, lanes, gs, tpb, sh.lg_ts);
            LW_LAUNCH_CHECK();
            return LW_OK;
        }
        default: return LW_E_INVALID_ARG;
    }
#undef LW_MM_DISPATCH
}

int spmm(int schedule, const lw_csr_t* A, const void* B, void* C, int64_t n, int64_t lanes,
         int64_t gs, int64_t tpb, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (A->rows == 0 || n == 0) return LW_OK;
    if (schedule == LW_MERGE_PATH && (!ws || ws_bytes < spmm_wo_workspace(lanes, n)))
        return LW_E_WORKSPACE;
    if (lanes < 1 || ceil_div(lanes << 5, MM_NT) > 0x7fffffffLL) return LW_E_UNSUPPORTED;
    const bool o32 = A->offset_bits == 32;
    if (A->dtype == LW_F32)
        return o32 ? spmm_typed<int32_t, float>(schedule, A, B, C, n, lanes, gs, tpb, ws, s)
                   : spmm_typed<int64_t, float>(schedule, A, B, C, n, lanes, gs, tpb, ws, s);
    return o32 ? spmm_typed<int32_t, double>(schedule, A, B, C, n, lanes, gs, tpb, ws, s)
               : spmm_typed<int64_t, double>(schedule, A, B, C, n, lanes, gs, tpb, ws, s);
}

}  // namespace lw
