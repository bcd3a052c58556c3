// spmv_work_oriented.cu — work_oriented (merge-path) schedule.
//
// Schedule (reference schedules.py:63-110): the merge path over
// (row boundaries x atoms) has rows+nnz items; lane k of P owns diagonals
// [min(k*items, total), min((k+1)*items, total)) with items = ceil(total/P), i.e.
// exactly merge_path_partition(ts, P). Ties consume the row boundary first, so an
// empty row costs one item (schedules.py:81).
//
// Device mapping. A lane is one CTA (the merge path is "searched per CTA",
// BASELINE.json north star); three stream-ordered kernels:
//  1. k_merge_path_search: one binary search per chunk boundary over off[t]+t —
//     the same search lw_merge_path_partition exports, bit-exact with
//     schedules.merge_path_partition (with one chunk per lane the boundaries are
//     exactly the partition at P lanes).
//  2. k_wo_chunk: the even-share SpMV of each lane's slice, chunk by chunk
//     (details above the kernel); the lane's trailing partial row becomes its
//     carry-out (reference _fast.py:46-52).
//  3. k_carry_fixup: adds carry-outs to their rows in lane order — the device
//     form of the serial fix-up kernels.py:90-91 / fixup_combine
//     (executor.py:212-221). Runs of carries into one row are summed in order,
//     so results are run-to-run reproducible (no float atomics).
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "lw_common.cuh"

namespace lw {

// Lane geometry (every dtype) and fp32 chunk geometry: a chunk is at most WO_S
// merge-path items (rows + atoms) and its atoms sit in an 8-aligned window of
// WO_W atoms (fp64 chunks are smaller, WoCfg<double>).
#ifndef LW_WO_W
#define LW_WO_W 4096
#endif
constexpr int WO_W = LW_WO_W;
constexpr int WO_S = WO_W - 16;
#ifndef LW_WO_PDL   // A/B: chunk and fix-up kernels as programmatic dependent launches
#define LW_WO_PDL 1
#endif
#ifndef LW_WO_WARP_SEARCH   // partitions of at most this many boundaries use the warp-cooperative search
#define LW_WO_WARP_SEARCH 12288
#endif
#ifndef LW_WO_BATCH   // A/B: batch the unpacked kernel's gathers like the packed one's
#define LW_WO_BATCH 0
#endif
constexpr unsigned WO_PHASE_PARTITION = 1, WO_PHASE_SPMV = 2, WO_PHASE_FIXUP = 4;

// threads x atoms-per-thread covering the window: one 32-byte col_idx load and
// one (fp32) or two (fp64) 32-byte value loads per thread. NT=512 x IPT=8 beat
// 256x16, 256x8 (W=2048) and 512x16 (W=8192) on C3 (kernel log).
template <class ValT>
struct WoCfg;
#ifndef LW_WO_NT
#define LW_WO_NT 512
#endif
// MAXR: register cap (fp64: 40 keeps 3 x 512 threads resident per SM; the
// allocator otherwise lands at 46-58). fp32 is left uncapped: it lands at 32
// (4 x 512, full occupancy) by itself, and a __maxnreg__(32) changes its code
// generation for the worse (0.992 -> 1.005 ms packed on C3).
// W / S: the dtype's chunk window (atoms) and chunk size (merge-path items). The
// LANE geometry stays WO_S for every dtype (lw_auto_lanes, probes and imbalance
// do not depend on the value type); fp64 cuts each lane into chunks of a 2048-atom
// window run by 256 threads (its 40-register, 3 x 512-thread geometry at 4096
// measured 1.349 ms on C3, 2048 x 256 1.30).
template <>
struct WoCfg<float> {
    static constexpr int NT = LW_WO_NT, IPT = WO_W / LW_WO_NT, MAXR = 0;   // uncapped
    static constexpr int W = WO_W, S = WO_S;
};
#ifndef LW_WO_MAXR64
#define LW_WO_MAXR64 40
#endif
#ifndef LW_WO_W64
#define LW_WO_W64 2048
#endif
#ifndef LW_WO_NT64
#define LW_WO_NT64 256
#endif
template <>
struct WoCfg<double> {
    static constexpr int NT = LW_WO_NT64, IPT = LW_WO_W64 / LW_WO_NT64, MAXR = LW_WO_MAXR64;
    // S: an exact fraction of the lane's WO_S items (2 chunks per lane at 2048,
    // none left over), at most W - 8 so the 8-aligned window holds the chunk
    static constexpr int W = LW_WO_W64, S = WO_S / (WO_W / LW_WO_W64);
};
static_assert(WoCfg<double>::S + 8 <= WoCfg<double>::W && WoCfg<double>::S <= WO_S,
              "fp64 chunks within the lane geometry");
inline int wo_chunk_items(int dtype) { return dtype == LW_F32 ? WoCfg<float>::S : WoCfg<double>::S; }

// ---- 1. partition ---------------------------------------------------------
// Boundary b of lane l = b / J, chunk j = b % J sits on diagonal
// min(l*items + min(j*S, items), total); with J = 1 this is exactly
// schedules.merge_path_partition's min(k*items, total).
__device__ __forceinline__ int64_t wo_bound_diag(int64_t b, int64_t J, int64_t items, int64_t S,
                                                 int64_t total) {
    const int64_t l = J == 1 ? b : b / J, j = b - l * J;
    return min(l * items + min(j * S, items), total);
}

template <class OffT>
__global__ void k_merge_path_search(const OffT* __restrict__ off, int64_t rows, int64_t nnz,
                                    int64_t n_bounds, int64_t J, int64_t items, int64_t S,
                                    int64_t* __restrict__ out_tile,
                                    int64_t* __restrict__ out_coords,
                                    unsigned* __restrict__ ticket = nullptr) {
    if (LW_WO_PDL) pdl_trigger();   // the chunk kernel may launch; it waits for these results
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ticket && k == 0) *ticket = 0u;   // the carry fix-up's CTA counter
    if (k >= n_bounds) return;
    const int64_t d = wo_bound_diag(k, J, items, S, rows + nnz);
    int64_t lo = max((int64_t)0, d - nnz), hi = min(d, rows);
    // greatest t with off[t] <= d - t  (off[t]+t strictly increasing)
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (ld_off(off + mid) <= d - mid) lo = mid;
        else hi = mid - 1;
    }
    if (out_tile) out_tile[k] = lo;
    if (out_coords) {
        out_coords[2 * k] = lo;
        out_coords[2 * k + 1] = d - lo;
    }
}

// Warp-cooperative form of the same search, for launches with few boundaries
// (C1/C2/C4 sizes: a few thousand), where the per-thread binary search is a chain
// of ~24 dependent L2 round trips and nothing else runs: each round the warp
// probes 32 points of the remaining range and keeps the gap between the last
// true and the first false probe (off[t] + t is strictly increasing, so the true
// probes are a prefix), ~5 rounds instead of 24. Same result as the binary search
// (the greatest t with off[t] <= d - t). With many boundaries (C3: 68.7 K) the 32x
// probes make it request-bound, so launch_search keeps the per-thread search there.
template <class OffT>
__device__ __forceinline__ int64_t mp_search_warp(const OffT* __restrict__ off, int64_t d, int64_t rows,
                                                  int64_t nnz, int lane) {
    int64_t lo = max((int64_t)0, d - nnz), hi = min(d, rows);
    while (lo < hi) {
        const int64_t span = hi - lo;
        const int64_t p = lo + ((int64_t)(lane + 1) * span + 31) / 32;   // in (lo, hi], p of lane 31 = hi
        const unsigned m = __ballot_sync(0xffffffffu, ld_off(off + p) <= d - p);
        const int k = __popc(m);
        if (k == 32) return hi;
        hi = lo + ((int64_t)(k + 1) * span + 31) / 32 - 1;                // before the first false probe
        if (k) lo = lo + ((int64_t)k * span + 31) / 32;                   // the last true probe
    }
    return lo;
}

template <class OffT>
__global__ void k_merge_path_search_warp(const OffT* __restrict__ off, int64_t rows, int64_t nnz,
                                         int64_t n_bounds, int64_t J, int64_t items, int64_t S,
                                         int64_t* __restrict__ out_tile,
                                         int64_t* __restrict__ out_coords,
                                         unsigned* __restrict__ ticket = nullptr) {
    if (LW_WO_PDL) pdl_trigger();
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & (kWarp - 1);
    if (ticket && k == 0 && lane == 0) *ticket = 0u;
    if (k >= n_bounds) return;   // warp-uniform
    const int64_t d = wo_bound_diag(k, J, items, S, rows + nnz);
    const int64_t t = mp_search_warp(off, d, rows, nnz, lane);
    if (lane == 0) {
        if (out_tile) out_tile[k] = t;
        if (out_coords) {
            out_coords[2 * k] = t;
            out_coords[2 * k + 1] = d - t;
        }
    }
}

// ---- 2. chunked even-share SpMV -------------------------------------------------
// One CTA per lane. A lane's slice of the merge path is cut into chunks of at
// most WO_S items; chunk boundaries come from the partition kernel, so every
// chunk's atoms [a0, a1) and completed rows [t0, t1) are known up front. Per
// chunk:
//   1. thread t owns the IPT consecutive atoms base + IPT*t ... of the 8-aligned
//      window over [a0, a1) and fetches their col_idx / values with 32-byte
//      vector loads (whole sectors, the warp reads contiguous bytes), issues its
//      first row-end load, then all IPT gathers of x at once;
//   2. the chunk's row ends are staged in shared memory and marked in a bit
//      mask of segment heads;
//   3. a block-wide segmented inclusive scan (thread-serial over IPT atoms,
//      warp shuffles, then across warps) turns products into running row sums;
//      each completed row reads its sum at its last atom and is written once
//      (coalesced; empty rows get 0);
//   4. the trailing partial row is carried to the lane's next chunk, and the
//      lane's final partial becomes its carry-out.
// The scan runs in the value precision: a chunk's partial sums pass through at
// most IPT + 5 + NT/32 additions, far inside the 1e-5 (fp32) bound; partials
// that cross chunks are carried in fp64.
template <int NT>
struct WoScan {
    int has[NT / kWarp];
    double val[NT / kWarp];
};

template <class ValT>
struct WoSmem {
    // row ends are window positions (< W <= 4096): 16 bits each, which leaves
    // 32 KB more of each SM's unified L1/shared array to cache x (-8% time on C3)
    static constexpr int W = WoCfg<ValT>::W, S = WoCfg<ValT>::S;
    static constexpr size_t end_off = 0;                                   // uint16[S]
    static constexpr size_t seg_off = (end_off + sizeof(uint16_t) * S + 15) / 16 * 16;  // ValT[W]
    static constexpr size_t flag_off = seg_off + sizeof(ValT) * W;         // uint32[W/32+2]
    static constexpr size_t bytes = flag_off + sizeof(uint32_t) * (W / 32 + 2);
};

// ---- fused all-gather output (power iteration over NVLink) -------------------------
// Every row the SpMV produces is also stored into the next-x buffer of every rank:
// either through the NVLS multicast address (one multimem.st reaches all GPUs on
// the NVSwitch) or, without multicast, one P2P store per peer buffer. Row t of
// this rank's shard lands at element base + t of each buffer.
constexpr int LW_MAX_PEERS = 8;
struct PeerOut {
    int32_t n;                      // peer buffers (ignored when mc is set)
    int64_t base;                   // global row of this shard's first row
    uint64_t ptr[LW_MAX_PEERS];     // peer buffer base addresses (UVA, P2P-mapped)
    uint64_t mc;                    // multicast base address, 0 = none
};

template <bool SP = false>   // SP: peer bases from shared memory (a runtime-bounded loop)
__device__ __forceinline__ void peer_store(const PeerOut& po, const uint64_t* sptr, int64_t row, float v) {
    if (po.mc) {
        asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(po.mc + (uint64_t)(po.base + row) * 4),
                     "f"(v) : "memory");
        return;
    }
    if constexpr (SP) {
#pragma unroll 1
        for (int p = 0; p < po.n; ++p) reinterpret_cast<float*>(sptr[p])[po.base + row] = v;
    } else {
#pragma unroll   // constant indices: the pointers stay in the parameter bank (no stack copy)
        for (int p = 0; p < LW_MAX_PEERS; ++p)
            if (p < po.n) reinterpret_cast<float*>(po.ptr[p])[po.base + row] = v;
    }
}
template <bool SP = false>   // SP: peer bases from shared memory (a runtime-bounded loop)
__device__ __forceinline__ void peer_store(const PeerOut& po, const uint64_t* sptr, int64_t row, double v) {
    if (po.mc) {
        asm volatile("multimem.st.relaxed.sys.global.f64 [%0], %1;" ::"l"(po.mc + (uint64_t)(po.base + row) * 8),
                     "d"(v) : "memory");
        return;
    }
    if constexpr (SP) {
#pragma unroll 1
        for (int p = 0; p < po.n; ++p) reinterpret_cast<double*>(sptr[p])[po.base + row] = v;
    } else {
#pragma unroll
        for (int p = 0; p < LW_MAX_PEERS; ++p)
            if (p < po.n) reinterpret_cast<double*>(po.ptr[p])[po.base + row] = v;
    }
}

// 8 consecutive col_idx / values with 32-byte loads (sm_100 .v8.b32 / .v4.b64)
__device__ __forceinline__ void ld8_col(const int32_t* p, int32_t* c) {
    const uint64_t pol = policy_evict_first();
    asm(
        "ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
        : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]),
          "=r"(c[7])
        : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld8_val(const float* p, float* v) {
    const uint64_t pol = policy_evict_first();
    uint32_t r[8];
    asm(
        "ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "l"(p), "l"(pol));
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __uint_as_float(r[k]);
}
__device__ __forceinline__ void ld8_val(const double* p, double* v) {
    const uint64_t pol = policy_evict_first();
    unsigned long long r[8];
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=l"(r[0]), "=l"(r[1]), "=l"(r[2]), "=l"(r[3]) : "l"(p), "l"(pol));
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b64 {%0,%1,%2,%3}, [%4], %5;"
                 : "=l"(r[4]), "=l"(r[5]), "=l"(r[6]), "=l"(r[7]) : "l"(p + 4), "l"(pol));
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __longlong_as_double((long long)r[k]);
}

// 4 consecutive col_idx / values with 16-byte (fp32) or 32-byte (fp64) loads
__device__ __forceinline__ void ld4_col(const int32_t* p, int32_t* c) {
    const uint64_t pol = policy_evict_first();
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld4_val(const float* p, float* v) {
    const uint64_t pol = policy_evict_first();
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
        : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void ld4_val(const double* p, double* v) {
    const uint64_t pol = policy_evict_first();
    unsigned long long r[4];
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b64 {%0,%1,%2,%3}, [%4], %5;"
        : "=l"(r[0]), "=l"(r[1]), "=l"(r[2]), "=l"(r[3]) : "l"(p), "l"(pol));
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __longlong_as_double((long long)r[k]);
}
// a thread's IPT consecutive (col, val) with the widest loads that fit
template <int IPT, class ValT>
__device__ __forceinline__ void ld_atoms(const int32_t* col, const ValT* val, int32_t* c, ValT* v) {
    if constexpr (IPT % 8 == 0) {
#pragma unroll
        for (int h = 0; h < IPT / 8; ++h) { ld8_col(col + 8 * h, c + 8 * h); ld8_val(val + 8 * h, v + 8 * h); }
    } else {
        static_assert(IPT % 4 == 0, "IPT must be a multiple of 4");
#pragma unroll
        for (int h = 0; h < IPT / 4; ++h) { ld4_col(col + 4 * h, c + 4 * h); ld4_val(val + 4 * h, v + 4 * h); }
    }
}

// fp64 running sums s_seg are stored transposed: window position pos lives at
// (pos % IPT) * NT + pos / IPT, so thread t writes its IPT consecutive sums with
// IPT scalar stores at t, NT + t, ... — every warp store is 32 consecutive
// doubles, conflict-free. Row-major with 16-byte stores puts a quarter warp's 8
// stores in 2 bank groups (53 M conflict wavefronts per C3 launch); transposed,
// fp64 C3 goes 1.588 -> 1.478 ms. fp32 stays row-major with float4 stores: its
// 2-way conflicts (9 M wavefronts) cost less than the 8 scalar stores
// (1.005 -> 1.026 ms packed, DESIGN.md kernel log).
template <class ValT>
struct SegT {
    static constexpr bool on = sizeof(ValT) == 8;
};
template <class ValT, int NT, int IPT>
__device__ __forceinline__ int seg_at(int pos) {
    if constexpr (!SegT<ValT>::on) return pos;
    else return (int)(((unsigned)pos % IPT) * NT + (unsigned)pos / IPT);
}
template <int NT, int IPT>
__device__ __forceinline__ void store_run(float* seg, int pos, const float* v) {
    float4* d = reinterpret_cast<float4*>(seg + pos);
#pragma unroll
    for (int h = 0; h < IPT / 4; ++h) d[h] = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
}
template <int NT, int IPT>
__device__ __forceinline__ void store_run(double* seg, int pos, const double* v) {
#pragma unroll
    for (int k = 0; k < IPT; ++k) seg[k * NT + (unsigned)pos / IPT] = v[k];
}

// Hot-x packed gather (lw_hotx_build relabels the most gathered columns c to
// slot | 0x80000000 and lw_spmv_work_oriented_hotx packs xh[slot] = x[c] per
// call): the packed hot values, 8 per 32-byte sector, are kept in L1
// (evict_last) and every other gather bypasses L1 (no_allocate), so the cold
// misses cannot evict the hot lines. Both loads stay on the read-only path.
__device__ __forceinline__ float ld_hotx(const float* x, const float* xh, int32_t c) {
    float v;
    if (c < 0)
        LW_LDASM("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(xh + (c & 0x7fffffff)));
    else
        LW_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(v) : "l"(x + c), "l"(policy_evict_last()));
    return v;
}
__device__ __forceinline__ double ld_hotx(const double* x, const double* xh, int32_t c) {
    double v;
    if (c < 0)
        LW_LDASM("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(xh + (c & 0x7fffffff)));
    else
        LW_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(x + c), "l"(policy_evict_last()));
    return v;
}

template <class OffT, class ValT, bool PROBE, bool VEC, bool PEERS, bool HOT>
__device__ __forceinline__ void wo_chunk_body(Csr<OffT, ValT> A, const ValT* __restrict__ x, ValT* __restrict__ y,
                                              int64_t items, int64_t J, const int64_t* __restrict__ bound_tile,
                                              int64_t* __restrict__ carry_tile, double* __restrict__ carry_val,
                                              Probe probe, PeerOut po, const ValT* __restrict__ xh) {
    constexpr int NT = WoCfg<ValT>::NT, IPT = WoCfg<ValT>::IPT;
    constexpr int W = WoCfg<ValT>::W, S = WoCfg<ValT>::S;
    static_assert(NT * IPT == W, "window must be NT*IPT atoms");
    using SM = WoSmem<ValT>;
    extern __shared__ __align__(16) unsigned char sm[];
    uint16_t* s_end = reinterpret_cast<uint16_t*>(sm + SM::end_off);
    static_assert(W <= 65536, "window positions must fit 16 bits");
    ValT* s_seg = reinterpret_cast<ValT*>(sm + SM::seg_off);
    uint32_t* s_flag = reinterpret_cast<uint32_t*>(sm + SM::flag_off);
    __shared__ WoScan<NT> scan;
    __shared__ uint64_t s_peer[PEERS && HOT ? LW_MAX_PEERS : 1];   // peer bases (packed variant)
    if (PEERS && HOT && threadIdx.x == 0) {
#pragma unroll   // constant indices keep the parameter struct in the constant bank
        for (int p = 0; p < LW_MAX_PEERS; ++p) s_peer[p] = po.ptr[p];
    }

    if (LW_WO_PDL) pdl_wait();   // chunk bounds and the packed hot x come from the partition launch
    const int tid = threadIdx.x, lane = tid & (kWarp - 1), warp = tid >> 5;
    const int64_t l = blockIdx.x;
    const int64_t total = A.rows + A.nnz;
    const int64_t lane_d0 = l * items;
    int64_t run_row = -1;    // lane-level partial carried across chunks
    double run_val = 0.0;
    bool run_has = false;
    int64_t lane_atoms = 0;

    for (int64_t jc = 0; jc < J; ++jc) {
        const int64_t d0 = min(lane_d0 + min(jc * S, items), total);
        const int64_t d1 = min(lane_d0 + min((jc + 1) * S, items), total);
        if (d0 >= d1) break;
        const int64_t t0 = bound_tile[l * J + jc], t1 = bound_tile[l * J + jc + 1];
        const int64_t a0 = d0 - t0;
        const int n_rows = (int)(t1 - t0), n_atoms = (int)((d1 - t1) - a0);
        const int64_t base = a0 & ~(int64_t)7;
        const int w0 = (int)(a0 - base);     // window position of a0
        const int w1 = w0 + n_atoms;         // one past the last atom
        lane_atoms += n_atoms;

        // zero the head mask (the previous chunk's readers finished at its last barrier)
        if (tid <= W / 32 + 1) s_flag[tid] = 0u;

        // 1. every global load of the chunk is issued before its first use
        const int pos = IPT * tid;           // window position of my first atom
        const int64_t g = base + pos;
        ValT p[IPT];
        const bool row0 = tid < n_rows;
        int32_t e0 = 0;
        {
            int32_t c[IPT];
            ValT v[IPT];
#pragma unroll
            for (int k = 0; k < IPT; ++k) {
                // atoms past the window still issue their (discarded) gather: point it at
                // x[0] (L1-allocating) or, packed, at hot slot 0 (kept in L1), never at a
                // no_allocate load that would cost an L2 request
                c[k] = HOT ? (int32_t)0x80000000 : 0;
                v[k] = (ValT)0;
            }
            if (pos < w1) {
                if (VEC && g + IPT <= A.nnz) {
                    ld_atoms<IPT>(A.col + g, A.val + g, c, v);
                } else {
#pragma unroll
                    for (int k = 0; k < IPT; ++k)
                        if (g + k < A.nnz) { c[k] = ld_stream(A.col + g + k); v[k] = ld_stream(A.val + g + k); }
                }
            }
            if (row0) e0 = (int32_t)(ld_off(A.off + t0 + 1 + tid) - base);
            if constexpr (HOT || LW_WO_BATCH) {
                // all IPT gathers issued back to back, unconditionally (every c[k] is
                // a valid column, x[0] or hot slot 0), before the first product consumes one
#pragma unroll
                for (int k = 0; k < IPT; ++k) {
                    if constexpr (HOT) p[k] = ld_hotx(x, xh, c[k]);
                    else p[k] = ld_gather(x + c[k]);
                }
            }
#pragma unroll
            for (int k = 0; k < IPT; ++k) {
                const bool in = pos + k >= w0 && pos + k < w1;
                if constexpr (HOT || LW_WO_BATCH) p[k] = in ? v[k] * p[k] : (ValT)0;
                else p[k] = in ? v[k] * ld_gather(x + c[k]) : (ValT)0;
            }
        }

        // 2. row ends + segment-head bit mask
        __syncthreads();
        if (row0) {
            s_end[tid] = e0;
            if (e0 < W) atomicOr(&s_flag[e0 >> 5], 1u << (e0 & 31));
        }
        for (int i = tid + NT; i < n_rows; i += NT) {   // chunks with more rows than threads
            const int e = (int)(ld_off(A.off + t0 + 1 + i) - base);
            s_end[i] = e;
            if (e < W) atomicOr(&s_flag[e >> 5], 1u << (e & 31));
        }
        __syncthreads();

        // 3. segmented scan: thread-serial, then warp shuffles, then across warps
        uint32_t fl;
        {
            const uint64_t two = ((uint64_t)s_flag[(pos >> 5) + 1] << 32) | s_flag[pos >> 5];
            fl = (uint32_t)(two >> (pos & 31)) & (uint32_t)((1ull << IPT) - 1ull);
        }
        bool has = fl != 0u;
        ValT run = (ValT)0;
#pragma unroll
        for (int k = 0; k < IPT; ++k) run = ((fl >> k) & 1u) ? p[k] : run + p[k];
#pragma unroll
        for (int d = 1; d < kWarp; d <<= 1) {
            const ValT ov = shfl_up(run, d);
            const int oh = shfl_up((int)has, d);
            if (lane >= d) {
                if (!has) run += ov;
                has = has || oh;
            }
        }
        if (lane == kWarp - 1) { scan.has[warp] = has; scan.val[warp] = (double)run; }
        __syncthreads();
        ValT wpre = (ValT)0;   // open segment entering my warp
        {
            bool h = false;
            for (int w = warp - 1; w >= 0 && !h; --w) {
                wpre += (ValT)scan.val[w];
                h = scan.has[w];
            }
        }
        ValT cin = shfl_up(run, 1);
        const int hin = shfl_up((int)has, 1);
        if (lane == 0) cin = wpre;
        else if (!hin) cin += wpre;
        {
            // running sums, stored with 16-byte vector stores (a thread's IPT
            // consecutive slots; scalar stores would be an 8-way bank conflict)
            ValT r = cin;
#pragma unroll
            for (int k = 0; k < IPT; ++k) {
                r = ((fl >> k) & 1u) ? p[k] : r + p[k];
                p[k] = r;
            }
            store_run<NT, IPT>(s_seg, pos, p);
        }
        __syncthreads();

        // 4. completed rows (coalesced), then the trailing partial
        for (int i = tid; i < n_rows; i += NT) {
            const int e = s_end[i];
            const int st = i ? s_end[i - 1] : w0;
            double v = e > st ? (double)s_seg[seg_at<ValT, NT, IPT>(e - 1)] : 0.0;
            if (i == 0 && run_has && run_row == t0) v += run_val;
            y[t0 + i] = (ValT)v;
            if (PEERS) peer_store<HOT>(po, s_peer, t0 + i, (ValT)v);   // smem bases: packed 1.24 -> 1.18 ms, unpacked 1.30 -> 1.50 (kept on the constant bank)
        }
        if (PROBE) {
            for (int w = tid; w < n_atoms; w += NT) {
                const int wp = w0 + w;
                int lo = 0, hi = n_rows;   // rows whose end <= wp come before the atom's row
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (s_end[mid] <= wp) lo = mid + 1;
                    else hi = mid;
                }
                probe_atom(probe, a0 + w, l, t0 + lo);
            }
        }
        {
            const int st = n_rows ? s_end[n_rows - 1] : w0;
            const bool tail = w1 > st;
            const double tv = tail ? (double)s_seg[seg_at<ValT, NT, IPT>(w1 - 1)] : 0.0;
            if (n_rows > 0) {
                run_row = t1; run_val = tv; run_has = tail;
            } else if (run_has && run_row == t1) {
                run_val += tv;
            } else {
                run_row = t1; run_val = tv; run_has = tail;
            }
        }
        if (jc + 1 < J) __syncthreads();   // s_end / s_seg / s_flag are rewritten by the next chunk
    }
    if (tid == 0) {
        const bool live = run_has && run_row >= 0 && run_row < A.rows;
        carry_tile[l] = live ? run_row : -1;
        carry_val[l] = live ? run_val : 0.0;
        if (PROBE && probe.lane_atoms) probe.lane_atoms[l] = lane_atoms;
    }
}

// The chunk kernel: fp32 with the allocator's own register choice (32), fp64
// capped at WoCfg<double>::MAXR (40; the peers variant 48) — see WoCfg.
#define LW_WO_PARAMS                                                                                  \
    Csr<OffT, ValT> A, const ValT *__restrict__ x, ValT *__restrict__ y, int64_t items, int64_t J,    \
        const int64_t *__restrict__ bound_tile, int64_t *__restrict__ carry_tile,                     \
        double *__restrict__ carry_val, Probe probe, PeerOut po, const ValT *__restrict__ xh
template <class OffT, class ValT, bool PROBE, bool VEC, bool PEERS = false, bool HOT = false>
__global__ void __launch_bounds__(WoCfg<ValT>::NT) k_wo_chunk(LW_WO_PARAMS) {
    wo_chunk_body<OffT, ValT, PROBE, VEC, PEERS, HOT>(A, x, y, items, J, bound_tile, carry_tile, carry_val,
                                                      probe, po, xh);
}
template <class OffT, class ValT, bool PROBE, bool VEC, bool PEERS = false, bool HOT = false>
__global__ void __launch_bounds__(WoCfg<ValT>::NT) __maxnreg__(PROBE ? 128 : WoCfg<double>::MAXR + (PEERS ? 8 : 0))
    k_wo_chunk64(LW_WO_PARAMS) {
    wo_chunk_body<OffT, ValT, PROBE, VEC, PEERS, HOT>(A, x, y, items, J, bound_tile, carry_tile, carry_val,
                                                      probe, po, xh);
}
#undef LW_WO_PARAMS
template <class OffT, class ValT, bool PROBE, bool VEC, bool PEERS = false, bool HOT = false>
constexpr auto wo_chunk_kernel() {
    if constexpr (sizeof(ValT) == 8) return &k_wo_chunk64<OffT, ValT, PROBE, VEC, PEERS, HOT>;
    else return &k_wo_chunk<OffT, ValT, PROBE, VEC, PEERS, HOT>;
}

// ---- 3. ordered carry fix-up -----------------------------------------------------
// Adds every lane's carry-out to its row (reference kernels.py:90-91: serial,
// in lane order). Carry rows are nondecreasing along the path with sentinels
// (-1) where a lane ended on a row boundary, so each row's carries form one
// contiguous run. Runs are summed by a segmented reduction, never by a walk:
// each CTA scans FX_NT consecutive carries (warp shuffles, then across warps);
// a run that starts and ends inside the CTA is added to y by its last carry's
// thread; the (at most two) run pieces that touch the CTA's edges are recorded
// and the last CTA to finish (atomic ticket) adds the runs that cross CTAs in
// path order. Every row is updated by exactly one thread, no float atomics:
// y is run-to-run reproducible, and a row spanning all 68 K lanes costs the
// same as any other (one scan step), where a per-row walk would be serial.
constexpr int FX_NT = 1024;
struct FixSeg {
    int64_t key;   // row, or -2 = empty slot
    double sum;
};

__device__ __forceinline__ int64_t fx_key(const int64_t* __restrict__ t, int64_t i, int64_t rows) {
    const int64_t r = t[i];
    return (r >= 0 && r < rows) ? r : -1;
}

template <class ValT, bool PEERS = false>
__global__ void __launch_bounds__(FX_NT)
    k_carry_fixup(const int64_t* __restrict__ carry_tile, const double* __restrict__ carry_val,
                  int64_t n, ValT* __restrict__ y, int64_t rows, unsigned* __restrict__ ticket,
                  FixSeg* __restrict__ segs, PeerOut po = PeerOut{}) {
    __shared__ double s_sum[FX_NT / kWarp];
    __shared__ int s_has[FX_NT / kWarp];
    __shared__ bool s_last;
    if (LW_WO_PDL) pdl_wait();   // carries come from the chunk kernel
    const int tid = threadIdx.x, lane = tid & (kWarp - 1), warp = tid >> 5;
    const int64_t c0 = (int64_t)blockIdx.x * FX_NT, c1 = min(c0 + FX_NT, n), i = c0 + tid;
    const bool in = i < c1;
    const int64_t key = in ? fx_key(carry_tile, i, rows) : -3;
    const double v = in && key >= 0 ? carry_val[i] : 0.0;
    // neighbours' keys from the warp, the warp-edge ones from memory
    int64_t prev = shfl_up(key, 1), next = __shfl_down_sync(0xffffffffu, key, 1);
    if (lane == 0) prev = i > 0 && in ? fx_key(carry_tile, i - 1, rows) : -4;
    if (lane == kWarp - 1 || i + 1 >= c1) next = i + 1 < n ? fx_key(carry_tile, i + 1, rows) : -5;
    // head: first carry of its run; the CTA's first carry is a head only if the
    // run really starts there
    const bool head = in && (i == 0 || prev != key);
    const bool brk = in && (i == c0 || head);   // scan segment boundary
    const bool tail = in && next != key;
    if (tid < 2 && gridDim.x > 1) segs[2 * blockIdx.x + tid] = FixSeg{-2, 0.0};

    // segmented inclusive scan of v (segments start at brk) + "a head in my segment"
    double run = v;
    bool has = brk, hh = head;   // hh: the segment's start is a true run head
    for (int d = 1; d < kWarp; d <<= 1) {
        const double ov = shfl_up(run, d);
        const int oh = shfl_up((int)has, d);
        const int ohh = shfl_up((int)hh, d);
        if (lane >= d && !has) {
            run += ov;
            has = oh;
            hh = ohh;
        }
    }
    if (lane == kWarp - 1) { s_sum[warp] = run; s_has[warp] = has ? (hh ? 2 : 1) : 0; }
    __syncthreads();
    if (!has) {   // my segment started in an earlier warp
        for (int w = warp - 1; w >= 0; --w) {
            run += s_sum[w];
            if (s_has[w]) { hh = s_has[w] == 2; break; }
        }
    }
    const bool last_in_cta = in && i == c1 - 1;
    if (in && key >= 0) {
        if (tail && hh) {                       // the whole run is inside this CTA
            const ValT out = (ValT)((double)y[key] + run);
            y[key] = out;
            if (PEERS) peer_store(po, po.ptr, key, out);
        } else if (tail && !hh) {               // piece that started before this CTA
            segs[2 * blockIdx.x] = FixSeg{key, run};
        } else if (last_in_cta) {               // piece that continues into the next CTA
            segs[2 * blockIdx.x + (hh ? 1 : 0)] = FixSeg{key, run};
        }
    }
    // one CTA: every run started and ended inside it (no pieces, no merge)
    if (gridDim.x == 1) return;
    // the last CTA to finish adds the runs that cross CTAs, in path order
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // Stage the pieces through shared memory in passes of FX_NT slots, compacted
    // (empty slots dropped, path order kept); the last piece of every run then sums
    // its run's pieces in path order — the same additions, in the same order, as a
    // serial walk (round 1's single-thread merge cost 37 us at C5's 276 K lanes, one
    // dependent y round trip per run) — and updates y. A run still open at the end
    // of a pass is carried into the next.
    __shared__ int64_t s_key[FX_NT];
    __shared__ double s_val[FX_NT];
    __shared__ int s_wcnt[FX_NT / kWarp];
    __shared__ int64_t s_ckey;    // run carried over from the previous pass (-2: none)
    __shared__ double s_cacc;
    if (tid == 0) { s_ckey = -2; s_cacc = 0.0; }
    const int64_t ns = 2 * (int64_t)gridDim.x;
    for (int64_t base = 0; base < ns; base += FX_NT) {
        const int64_t k = base + tid;
        const int64_t kk = k < ns ? __ldcg(&segs[k].key) : -2;
        const double kv = k < ns ? __ldcg(&segs[k].sum) : 0.0;
        const bool valid = kk >= 0;
        const unsigned bal = __ballot_sync(0xffffffffu, valid);
        if (lane == 0) s_wcnt[warp] = __popc(bal);
        __syncthreads();   // (the previous pass is done with s_key / s_val / the carry)
        const int64_t ckey = s_ckey;
        const double cacc = s_cacc;
        int off = 0, m = 0;
        for (int w = 0; w < FX_NT / kWarp; ++w) {
            const int c = s_wcnt[w];
            off += w < warp ? c : 0;
            m += c;
        }
        if (valid) {
            const int p = off + __popc(bal & ((1u << lane) - 1u));
            s_key[p] = kk;
            s_val[p] = kv;
        }
        __syncthreads();
        const bool more = base + FX_NT < ns;   // a later pass may continue the last run
        if (tid < m) {
            const int64_t key = s_key[tid];
            const bool end = tid + 1 < m ? s_key[tid + 1] != key : !more;
            const bool carry_out = tid == m - 1 && more;
            double acc = 0.0;
            if (end || carry_out) {
                int st = tid;
                while (st > 0 && s_key[st - 1] == key) --st;
                acc = (st == 0 && ckey == key) ? cacc : 0.0;
                for (int j = st; j <= tid; ++j) acc += s_val[j];
                if (end) {
                    const ValT out = (ValT)((double)y[key] + acc);
                    y[key] = out;
                    if (PEERS) peer_store(po, po.ptr, key, out);
                }
            }
            if (tid == m - 1) { s_ckey = carry_out ? key : -2; s_cacc = carry_out ? acc : 0.0; }
        }
        // a carried run that this pass does not continue ends where it was carried
        // (an empty pass keeps it for the next one)
        if (tid == 0 && ckey >= 0 && (m > 0 ? s_key[0] != ckey : !more)) {
            const ValT out = (ValT)((double)y[ckey] + cacc);
            y[ckey] = out;
            if (PEERS) peer_store(po, po.ptr, ckey, out);
        }
    }
    __syncthreads();
    if (tid == 0) {
        *ticket = 0u;   // ready for the next launch on this workspace
    }
}

// ---- 4. hot-x pack: xh[slot] = x[hot_cols[slot]] (n_hot gathers per call) ----------------
template <class ValT>
__global__ void k_hot_pack(const ValT* __restrict__ x, const int32_t* __restrict__ hot_cols,
                           int32_t n_hot, ValT* __restrict__ xh) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n_hot) xh[i] = x[hot_cols[i]];
}

// The partition search and the hot-x pack are independent; one launch runs both
// (blocks [0, nsb) search, the rest pack), so the packed path adds no launch.
template <class OffT, class ValT>
__global__ void k_search_pack(const OffT* __restrict__ off, int64_t rows, int64_t nnz,
                              int64_t n_bounds, int64_t J, int64_t items, int64_t S,
                              int64_t* __restrict__ out_tile, unsigned nsb,
                              const ValT* __restrict__ x, const int32_t* __restrict__ hot_cols,
                              int32_t n_hot, ValT* __restrict__ xh, unsigned* __restrict__ ticket) {
    if (LW_WO_PDL) pdl_trigger();   // the chunk kernel may launch; it waits for these results
    if (blockIdx.x == 0 && threadIdx.x == 0) *ticket = 0u;
    if (blockIdx.x >= nsb) {
        const int i = (int)(blockIdx.x - nsb) * blockDim.x + threadIdx.x;
        if (i < n_hot) xh[i] = x[hot_cols[i]];
        return;
    }
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_bounds) return;
    const int64_t d = wo_bound_diag(k, J, items, S, rows + nnz);
    int64_t lo = max((int64_t)0, d - nnz), hi = min(d, rows);
    while (lo < hi) {   // greatest t with off[t] <= d - t, as k_merge_path_search
        const int64_t mid = (lo + hi + 1) >> 1;
        if (ld_off(off + mid) <= d - mid) lo = mid;
        else hi = mid - 1;
    }
    out_tile[k] = lo;
}

// ---- host side -------------------------------------------------------------------
struct WoPlan {
    int64_t total, lanes, items, J;
};

// lanes: the schedule's (auto: one WO_S-item lane per chunk of the fp32 geometry,
// for every dtype); J: chunks of at most `chunk` items per lane (the dtype's S)
static WoPlan wo_plan(int64_t rows, int64_t nnz, int64_t lanes, int64_t chunk = WO_S) {
    WoPlan p{};
    p.total = rows + nnz;
    if (lanes <= 0) lanes = p.total > 0 ? ceil_div(p.total, WO_S) : 1;
    p.lanes = lanes;
    p.items = p.total > 0 ? ceil_div(p.total, lanes) : 0;
    p.J = p.items > 0 ? ceil_div(p.items, chunk) : 1;
    return p;
}

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// carry slots: one per lane
static size_t wo_carries(const WoPlan& p) { return (size_t)p.lanes; }

// Workspace: chunk-boundary tiles, carry rows, carry values, the fix-up's
// ticket + edge pieces (2 per fix-up CTA); the hot-x variant appends xh.
struct WoWs {
    int64_t* tiles;
    int64_t* c_tile;
    double* c_val;
    unsigned* ticket;
    FixSeg* segs;
    unsigned char* end;
};

static size_t wo_fix_bytes(const WoPlan& p) {
    const size_t blocks = (size_t)ceil_div((int64_t)wo_carries(p), (int64_t)FX_NT);
    return align_up(16 + 2 * (blocks > 0 ? blocks : 1) * sizeof(FixSeg), 256);
}

static WoWs wo_ws(const WoPlan& p, void* ws) {
    const size_t nb = (size_t)(p.lanes * p.J + 1), nc = wo_carries(p);
    unsigned char* w = (unsigned char*)ws;
    WoWs r{};
    r.tiles = (int64_t*)w;
    w += align_up(nb * 8, 256);
    r.c_tile = (int64_t*)w;
    w += align_up(nc * 8, 256);
    r.c_val = (double*)w;
    w += align_up(nc * 8, 256);
    r.ticket = (unsigned*)w;
    r.segs = (FixSeg*)(w + 16);
    w += wo_fix_bytes(p);
    r.end = w;
    return r;
}

size_t wo_workspace(int64_t rows, int64_t nnz, int64_t lanes, int dtype) {
    const WoPlan p = wo_plan(rows, nnz, lanes, wo_chunk_items(dtype));
    const size_t nb = (size_t)(p.lanes * p.J + 1), nc = wo_carries(p);
    return align_up(nb * 8, 256) + 2 * align_up(nc * 8, 256) + wo_fix_bytes(p);
}

template <class ValT, bool PEERS = false>
static int launch_fixup(const WoWs& w, int64_t n, ValT* y, int64_t rows, cudaStream_t s,
                        const PeerOut& po = PeerOut{}) {
    if (n <= 0) return LW_OK;
    if (LW_WO_PDL)
        LW_TRY(launch_pdl(k_carry_fixup<ValT, PEERS>, dim3((unsigned)ceil_div(n, (int64_t)FX_NT)), dim3(FX_NT), 0, s,
                          w.c_tile, w.c_val, n, y, rows, w.ticket, w.segs, po));
    else
        k_carry_fixup<ValT, PEERS><<<(unsigned)ceil_div(n, (int64_t)FX_NT), FX_NT, 0, s>>>(
            w.c_tile, w.c_val, n, y, rows, w.ticket, w.segs, po);
    LW_LAUNCH_CHECK();
    return LW_OK;
}

int64_t wo_lanes(int64_t rows, int64_t nnz, int64_t lanes) { return wo_plan(rows, nnz, lanes).lanes; }

template <class OffT>
static int launch_search(const OffT* off, int64_t rows, int64_t nnz, int64_t n_bounds, int64_t J,
                         int64_t items, int64_t S, int64_t* out_tile, int64_t* out_coords,
                         cudaStream_t s, unsigned* ticket = nullptr) {
    const int NT = 256;
    if (n_bounds <= LW_WO_WARP_SEARCH)
        k_merge_path_search_warp<OffT><<<ceil_div(n_bounds * kWarp, NT), NT, 0, s>>>(
            off, rows, nnz, n_bounds, J, items, S, out_tile, out_coords, ticket);
    else
        k_merge_path_search<OffT><<<ceil_div(n_bounds, NT), NT, 0, s>>>(off, rows, nnz, n_bounds, J, items,
                                                                     S, out_tile, out_coords, ticket);
    LW_LAUNCH_CHECK();
    return LW_OK;
}

// Tiles of the chunk boundaries of merge_path_partition(ts, lanes) with each lane
// cut into J chunks of at most S items (boundary b = lane*J + chunk, as for the
// SpMV chunk kernel; J = 1 gives the partition's coords[:, 0]), for the SpMM
// work_oriented kernel. tiles: device int64[lanes*J + 1].
int mp_bound_tiles(const lw_csr_t* A, int64_t lanes, int64_t J, int64_t S, int64_t* tiles,
                   cudaStream_t s) {
    const int64_t total = A->rows + A->nnz;
    const int64_t items = total > 0 ? ceil_div(total, lanes) : 0;
    if (A->offset_bits == 32)
        return launch_search<int32_t>((const int32_t*)A->row_offsets, A->rows, A->nnz, lanes * J + 1,
                                      J, items, S, tiles, nullptr, s);
    return launch_search<int64_t>((const int64_t*)A->row_offsets, A->rows, A->nnz, lanes * J + 1, J,
                                  items, S, tiles, nullptr, s);
}

int merge_path_partition(int64_t rows, int64_t nnz, const void* off, int bits, int64_t lanes,
                         int64_t* coords, cudaStream_t s) {
    if (lanes < 1 || rows < 0 || nnz < 0 || !coords || (!off && rows > 0)) return LW_E_INVALID_ARG;
    const int64_t total = rows + nnz;
    const int64_t items = total > 0 ? ceil_div(total, lanes) : 0;
    if (bits == 32)
        return launch_search<int32_t>((const int32_t*)off, rows, nnz, lanes + 1, 1, items, items,
                                      nullptr, coords, s);
    return launch_search<int64_t>((const int64_t*)off, rows, nnz, lanes + 1, 1, items, items, nullptr,
                                  coords, s);
}


template <class OffT, class ValT, bool PR, bool VEC, bool HOT = false>
static int launch_chunk(const Csr<OffT, ValT>& a, const ValT* x, ValT* y, const WoPlan& p,
                        const int64_t* tiles, int64_t* c_tile, double* c_val, const Probe& pr,
                        cudaStream_t s, const ValT* xh = nullptr) {
    auto kern = wo_chunk_kernel<OffT, ValT, PR, VEC, false, HOT>();
    constexpr size_t smem = WoSmem<ValT>::bytes;
    static bool attr = false;   // one-time opt-in above the 48 KB default
    if (!attr) {
        LW_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (const char* cv = getenv("LW_WO_CARVEOUT"))   // A/B runs only
            LW_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv)));
        attr = true;
    }
    if (LW_WO_PDL)
        LW_TRY(launch_pdl(kern, dim3((unsigned)p.lanes), dim3(WoCfg<ValT>::NT), smem, s, a, x, y, p.items, p.J,
                          tiles, c_tile, c_val, pr, PeerOut{}, xh));
    else
        kern<<<(unsigned)p.lanes, WoCfg<ValT>::NT, smem, s>>>(a, x, y, p.items, p.J, tiles, c_tile,
                                                             c_val, pr, PeerOut{}, xh);
    LW_LAUNCH_CHECK();
    return LW_OK;
}

template <class OffT, class ValT>
static int launch_wo(const lw_csr_t* A, const void* x, void* y, const WoPlan& p, void* ws,
                     const lw_probe_t* probe, unsigned phases, cudaStream_t s,
                     const int32_t* hot_cols = nullptr, int32_t n_hot = 0) {
    Csr<OffT, ValT> a{A->rows, A->cols, A->nnz, (const OffT*)A->row_offsets,
                      A->col_indices, (const ValT*)A->values};
    const size_t nb = (size_t)(p.lanes * p.J + 1);
    const WoWs W = wo_ws(p, ws);
    int64_t* tiles = W.tiles;
    int64_t* c_tile = W.c_tile;
    double* c_val = W.c_val;
    ValT* xh = (ValT*)W.end;   // hot-x variant only: packed hot values after the base workspace
    Probe pr{};
    if (probe) pr = Probe{probe->lane_atoms, probe->atom_lane, probe->atom_tile, probe->atom_visits};
    if (p.lanes > 0x7fffffff) return LW_E_UNSUPPORTED;
    // 32-byte vector loads need 32-byte aligned col_idx / values
    const bool vec = ((uintptr_t)A->col_indices % 32 == 0) && ((uintptr_t)A->values % 32 == 0);
    const int64_t n_carry = p.lanes;   // one carry per lane

    if ((phases & WO_PHASE_PARTITION) && hot_cols && n_hot > 0) {   // partition + hot-x pack
        const unsigned nsb = (unsigned)ceil_div((int64_t)nb, 256);
        const unsigned npb = (unsigned)ceil_div(n_hot, 256);
        k_search_pack<OffT, ValT><<<nsb + npb, 256, 0, s>>>(a.off, a.rows, a.nnz, (int64_t)nb, p.J, p.items,
                                                          WoCfg<ValT>::S, tiles, nsb, (const ValT*)x, hot_cols,
                                                          n_hot, xh, W.ticket);
        LW_LAUNCH_CHECK();
    } else if (phases & WO_PHASE_PARTITION) {
        int rc = launch_search<OffT>(a.off, a.rows, a.nnz, (int64_t)nb, p.J, p.items, WoCfg<ValT>::S, tiles,
                                     nullptr, s, W.ticket);
        if (rc) return rc;
    }
    if (phases & WO_PHASE_SPMV) {
        if (probe && pr.lane_atoms) LW_TRY(cudaMemsetAsync(pr.lane_atoms, 0, p.lanes * 8, s));
        const ValT* xv = (const ValT*)x;
        ValT* yv = (ValT*)y;
        const bool P = probe != nullptr;
        int rc = LW_OK;
        if (hot_cols) {   // packed hot x lives after the base workspace
            // (xh was packed by the partition phase's launch, k_search_pack)
            rc = vec ? launch_chunk<OffT, ValT, false, true, true>(a, xv, yv, p, tiles, c_tile, c_val, pr, s, xh)
                     : launch_chunk<OffT, ValT, false, false, true>(a, xv, yv, p, tiles, c_tile, c_val, pr, s, xh);
        } else if (P) rc = vec ? launch_chunk<OffT, ValT, true, true>(a, xv, yv, p, tiles, c_tile, c_val, pr, s)
                        : launch_chunk<OffT, ValT, true, false>(a, xv, yv, p, tiles, c_tile, c_val, pr, s);
        else   rc = vec ? launch_chunk<OffT, ValT, false, true>(a, xv, yv, p, tiles, c_tile, c_val, pr, s)
                        : launch_chunk<OffT, ValT, false, false>(a, xv, yv, p, tiles, c_tile, c_val, pr, s);
        if (rc) return rc;
        LW_LAUNCH_CHECK();
    }
    if (phases & WO_PHASE_FIXUP) {
        int rc = launch_fixup<ValT>(W, n_carry, (ValT*)y, a.rows, s);
        if (rc) return rc;
    }
    return LW_OK;
}

// SpMV whose rows also land in every rank's next-x buffer (fused all-gather).
template <class OffT, class ValT, bool HOT>
static int launch_wo_peers(const lw_csr_t* A, const void* x, void* y, const WoPlan& p, void* ws,
                           const PeerOut& po, cudaStream_t s, const int32_t* hot_cols, int32_t n_hot) {
    Csr<OffT, ValT> a{A->rows, A->cols, A->nnz, (const OffT*)A->row_offsets, A->col_indices,
                      (const ValT*)A->values};
    const size_t nb = (size_t)(p.lanes * p.J + 1);
    const WoWs W = wo_ws(p, ws);
    int64_t* tiles = W.tiles;
    int64_t* c_tile = W.c_tile;
    double* c_val = W.c_val;
    if (p.lanes > 0x7fffffff) return LW_E_UNSUPPORTED;
    int rc = launch_search<OffT>(a.off, a.rows, a.nnz, (int64_t)nb, p.J, p.items, WoCfg<ValT>::S, tiles, nullptr, s,
                                 W.ticket);
    if (rc) return rc;
    const bool vec = ((uintptr_t)A->col_indices % 32 == 0) && ((uintptr_t)A->values % 32 == 0);
    constexpr size_t smem = WoSmem<ValT>::bytes;
    auto kern = vec ? wo_chunk_kernel<OffT, ValT, false, true, true, HOT>()
                    : wo_chunk_kernel<OffT, ValT, false, false, true, HOT>();
    ValT* xh = nullptr;
    if constexpr (HOT) {   // packed hot x after the base workspace, as in launch_wo
        xh = (ValT*)W.end;
        if (n_hot > 0) {
            k_hot_pack<ValT><<<(unsigned)ceil_div(n_hot, 256), 256, 0, s>>>((const ValT*)x, hot_cols, n_hot, xh);
            LW_LAUNCH_CHECK();
        }
    }
    static bool attr[2] = {false, false};
    if (!attr[vec]) {
        LW_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr[vec] = true;
    }
    kern<<<(unsigned)p.lanes, WoCfg<ValT>::NT, smem, s>>>(a, (const ValT*)x, (ValT*)y, p.items, p.J,
                                                         tiles, c_tile, c_val, Probe{}, po, xh);
    LW_LAUNCH_CHECK();
    return launch_fixup<ValT, true>(W, p.lanes, (ValT*)y, a.rows, s, po);
}

size_t wo_hotx_workspace(int64_t rows, int64_t nnz, int64_t lanes, int64_t n_hot, int dtype);

int spmv_work_oriented_peers(const lw_csr_t* A, const void* x, void* y, int64_t lanes, void* ws,
                             size_t ws_bytes, int32_t n_peers, const uint64_t* peer_ptrs,
                             uint64_t mc_ptr, int64_t row_base, cudaStream_t s,
                             const int32_t* hot_cols, int32_t n_hot) {
    if (n_peers < 0 || n_peers > LW_MAX_PEERS || (n_peers > 0 && !peer_ptrs) || row_base < 0 ||
        n_hot < 0 || (n_hot > 0 && !hot_cols))
        return LW_E_INVALID_ARG;
    const WoPlan p = wo_plan(A->rows, A->nnz, lanes, wo_chunk_items(A->dtype));
    if (A->rows == 0) return LW_OK;
    const bool hot = hot_cols != nullptr || n_hot > 0;
    const size_t need = hot ? wo_hotx_workspace(A->rows, A->nnz, lanes, n_hot, A->dtype)
                            : wo_workspace(A->rows, A->nnz, lanes, A->dtype);
    if (!ws || ws_bytes < need) return LW_E_WORKSPACE;
    PeerOut po{};
    po.n = n_peers;
    po.base = row_base;
    po.mc = mc_ptr;
    for (int i = 0; i < n_peers; ++i) po.ptr[i] = peer_ptrs[i];
    const bool o32 = A->offset_bits == 32;
    const int32_t* hc = hot_cols;
    if (hot) {
        if (A->dtype == LW_F32)
            return o32 ? launch_wo_peers<int32_t, float, true>(A, x, y, p, ws, po, s, hc, n_hot)
                       : launch_wo_peers<int64_t, float, true>(A, x, y, p, ws, po, s, hc, n_hot);
        return o32 ? launch_wo_peers<int32_t, double, true>(A, x, y, p, ws, po, s, hc, n_hot)
                   : launch_wo_peers<int64_t, double, true>(A, x, y, p, ws, po, s, hc, n_hot);
    }
    if (A->dtype == LW_F32)
        return o32 ? launch_wo_peers<int32_t, float, false>(A, x, y, p, ws, po, s, hc, 0)
                   : launch_wo_peers<int64_t, float, false>(A, x, y, p, ws, po, s, hc, 0);
    return o32 ? launch_wo_peers<int32_t, double, false>(A, x, y, p, ws, po, s, hc, 0)
               : launch_wo_peers<int64_t, double, false>(A, x, y, p, ws, po, s, hc, 0);
}

int spmv_work_oriented(const lw_csr_t* A, const void* x, void* y, int64_t lanes, void* ws,
                       size_t ws_bytes, const lw_probe_t* probe, unsigned phases,
                       cudaStream_t s) {
    const WoPlan p = wo_plan(A->rows, A->nnz, lanes, wo_chunk_items(A->dtype));
    if (A->rows == 0) return LW_OK;
    if (!ws || ws_bytes < wo_workspace(A->rows, A->nnz, lanes, A->dtype)) return LW_E_WORKSPACE;
    const bool o32 = A->offset_bits == 32;
    if (A->dtype == LW_F32)
        return o32 ? launch_wo<int32_t, float>(A, x, y, p, ws, probe, phases, s)
                   : launch_wo<int64_t, float>(A, x, y, p, ws, probe, phases, s);
    return o32 ? launch_wo<int32_t, double>(A, x, y, p, ws, probe, phases, s)
               : launch_wo<int64_t, double>(A, x, y, p, ws, probe, phases, s);
}

// Workspace of the hot-x variant: the plain one plus the packed hot values.
size_t wo_hotx_workspace(int64_t rows, int64_t nnz, int64_t lanes, int64_t n_hot, int dtype) {
    // at least one slot: atoms outside a chunk's window read (and discard) slot 0
    return wo_workspace(rows, nnz, lanes, dtype) + align_up((size_t)(n_hot > 0 ? n_hot : 1) * (dtype == LW_F32 ? 4 : 8), 256);
}

int spmv_work_oriented_hotx(const lw_csr_t* A, const int32_t* hot_cols, int32_t n_hot,
                            const void* x, void* y, int64_t lanes, void* ws, size_t ws_bytes,
                            unsigned phases, cudaStream_t s) {
    if (n_hot < 0 || (n_hot > 0 && !hot_cols)) return LW_E_INVALID_ARG;
    const WoPlan p = wo_plan(A->rows, A->nnz, lanes, wo_chunk_items(A->dtype));
    if (A->rows == 0) return LW_OK;
    if (!ws || ws_bytes < wo_hotx_workspace(A->rows, A->nnz, lanes, n_hot, A->dtype)) return LW_E_WORKSPACE;
    static const int32_t none = 0;   // any non-null marker selects the hot kernel when n_hot == 0
    const int32_t* hc = hot_cols ? hot_cols : &none;
    const bool o32 = A->offset_bits == 32;
    if (A->dtype == LW_F32)
        return o32 ? launch_wo<int32_t, float>(A, x, y, p, ws, nullptr, phases, s, hc, n_hot)
                   : launch_wo<int64_t, float>(A, x, y, p, ws, nullptr, phases, s, hc, n_hot);
    return o32 ? launch_wo<int32_t, double>(A, x, y, p, ws, nullptr, phases, s, hc, n_hot)
               : launch_wo<int64_t, double>(A, x, y, p, ws, nullptr, phases, s, hc, n_hot);
}

}  // namespace lw
