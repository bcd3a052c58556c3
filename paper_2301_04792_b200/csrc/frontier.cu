// frontier.cu — SSSP and BFS by frontier relaxation under the three schedules.
//
// Reference: kernels.sssp / sssp_pass / bfs (kernels.py:230-381), the numba
// loops _fast.sssp_relax / bfs_relax (_fast.py:147-170) and the schedule-driven
// pure passes (_sssp_pass_pure, _bfs_pass_pure, _walk_merge_path_atoms); the
// paper's Listing 5. One pass:
//   1. active = flatnonzero(in_frontier): ordered stream compaction (scan);
//   2. the frontier tile set: tiles = active vertices, atoms = their out-edges,
//      offsets = exclusive_prefix_sum(degrees) (kernels.py:271-275), on device;
//   3. every atom (edge u->v) relaxes v under the chosen schedule:
//        SSSP  nd = dist[u] + w;  old = atomicMin(dist[v], nd);  nd < old -> out[v]
//              (fp64 bit patterns of non-negative reals order like uint64, the
//              "order-preserving bit-pattern comparison" of executor.py:254-283)
//        BFS   depth[v] < 0 -> depth[v] = level+1, out[v]   (idempotent claim)
// A converged pass sequence reaches the unique least fixed point of
// d(v) = min over in-edges fl(d(u) + w), so distances are bit-identical to the
// reference's serial relaxation (and to Dijkstra) whatever the schedule.
#include <cstring>

#include "lw_common.cuh"

namespace lw {

int64_t group_auto_lanes(int64_t rows, int64_t gs, int64_t tpb);

// ---- device scan over n items produced by a functor (exclusive, int64) -----------------
constexpr int SC_NT = 512, SC_IPT = 4, SC_TILE = SC_NT * SC_IPT;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* s_warp, int64_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t o = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += o;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int64_t w = lane < SC_NT / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t o = __shfl_up_sync(0xffffffffu, w, d);
            if (lane >= d) w += o;
        }
        if (lane < SC_NT / 32) s_warp[lane] = w;   // inclusive warp totals
    }
    __syncthreads();
    const int64_t before = warp ? s_warp[warp - 1] : 0;
    if (total) *total = s_warp[SC_NT / 32 - 1];
    return before + x - v;
}

struct DegreeOf {   // degree of active vertex i
    const void* off;
    int bits;
    const int32_t* active;
    __device__ int64_t operator()(int64_t i) const {
        const int64_t u = active[i];
        if (bits == 32) {
            const int32_t* o = (const int32_t*)off;
            return (int64_t)__ldg(o + u + 1) - __ldg(o + u);
        }
        const int64_t* o = (const int64_t*)off;
        return __ldg(o + u + 1) - __ldg(o + u);
    }
};
struct FlagOf {
    const uint8_t* mask;
    __device__ int64_t operator()(int64_t i) const { return mask[i] != 0; }
};

template <class F>
__global__ void __launch_bounds__(SC_NT) k_scan_up(F f, int64_t n, int64_t* sums) {
    __shared__ int64_t s_warp[SC_NT / 32];
    const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_IPT;
    int64_t v = 0;
#pragma unroll
    for (int k = 0; k < SC_IPT; ++k)
        if (base + k < n) v += f(base + k);
    int64_t tot;
    block_excl_scan(v, s_warp, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// exclusive scan of m block sums in place (one CTA, chunks of SC_NT); sums[m] = total
__global__ void __launch_bounds__(SC_NT) k_scan_sums(int64_t* sums, int64_t m) {
    __shared__ int64_t s_warp[SC_NT / 32];
    int64_t carry = 0;
    for (int64_t c = 0; c < m; c += SC_NT) {
        const int64_t i = c + threadIdx.x;
        const int64_t v = i < m ? sums[i] : 0;
        int64_t tot;
        const int64_t ex = block_excl_scan(v, s_warp, &tot);
        __syncthreads();
        if (i < m) sums[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[m] = carry;
}

// out[i] = exclusive prefix (if out), out[n] = total; COMPACT: active[out_i] = i when f(i)
template <class F, bool COMPACT>
__global__ void __launch_bounds__(SC_NT)
    k_scan_down(F f, int64_t n, const int64_t* sums, int64_t* out, int32_t* compact) {
    __shared__ int64_t s_warp[SC_NT / 32];
    const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_IPT;
    int64_t v[SC_IPT], t = 0;
#pragma unroll
    for (int k = 0; k < SC_IPT; ++k) {
        v[k] = base + k < n ? f(base + k) : 0;
        t += v[k];
    }
    int64_t run = sums[blockIdx.x] + block_excl_scan(t, s_warp, nullptr);
#pragma unroll
    for (int k = 0; k < SC_IPT; ++k) {
        if (base + k < n) {
            if (out) out[base + k] = run;
            if (COMPACT && v[k]) compact[run] = (int32_t)(base + k);
        }
        run += v[k];
    }
}

static int64_t scan_blocks(int64_t n) { return n > 0 ? ceil_div(n, SC_TILE) : 1; }

template <class F, bool COMPACT>
static int scan_run(F f, int64_t n, int64_t* sums, int64_t* out, int32_t* compact, int64_t* total,
                    cudaStream_t s) {
    const int64_t nb = scan_blocks(n);
    if (n == 0) {
        if (out) LW_TRY(cudaMemsetAsync(out, 0, 8, s));
        if (total) LW_TRY(cudaMemsetAsync(total, 0, 8, s));
        return LW_OK;
    }
    k_scan_up<F><<<(unsigned)nb, SC_NT, 0, s>>>(f, n, sums);
    k_scan_sums<<<1, SC_NT, 0, s>>>(sums, nb);
    k_scan_down<F, COMPACT><<<(unsigned)nb, SC_NT, 0, s>>>(f, n, sums, out, compact);
    if (out) LW_TRY(cudaMemcpyAsync(out + n, sums + nb, 8, cudaMemcpyDeviceToDevice, s));
    if (total) LW_TRY(cudaMemcpyAsync(total, sums + nb, 8, cudaMemcpyDeviceToDevice, s));
    LW_LAUNCH_CHECK();
    return LW_OK;
}

// ---- fused frontier scan: active[] and frontier offsets fo[] in one sweep ---------------
// Item v contributes (mask[v] != 0, degree(v) if in the frontier): the exclusive
// prefix of the first gives v's slot in active[], of the second the offset of
// its out-edges in the frontier tile set. sums2 holds per-block pairs.
struct Pair {
    int64_t a, b;
};

__device__ __forceinline__ Pair block_excl_scan2(Pair v, Pair* s_warp, Pair* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Pair x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t oa = __shfl_up_sync(0xffffffffu, x.a, d);
        const int64_t ob = __shfl_up_sync(0xffffffffu, x.b, d);
        if (lane >= d) { x.a += oa; x.b += ob; }
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        Pair w = lane < SC_NT / 32 ? s_warp[lane] : Pair{0, 0};
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const int64_t oa = __shfl_up_sync(0xffffffffu, w.a, d);
            const int64_t ob = __shfl_up_sync(0xffffffffu, w.b, d);
            if (lane >= d) { w.a += oa; w.b += ob; }
        }
        if (lane < SC_NT / 32) s_warp[lane] = w;
    }
    __syncthreads();
    const Pair before = warp ? s_warp[warp - 1] : Pair{0, 0};
    if (total) *total = s_warp[SC_NT / 32 - 1];
    return Pair{before.a + x.a - v.a, before.b + x.b - v.b};
}

template <class OffT>
__device__ __forceinline__ Pair frontier_item(const uint8_t* mask, const OffT* off, int64_t v) {
    if (!mask[v]) return Pair{0, 0};
    return Pair{1, (int64_t)__ldg(off + v + 1) - (int64_t)__ldg(off + v)};
}

template <class OffT>
__global__ void __launch_bounds__(SC_NT)
    k_fscan_up(const uint8_t* __restrict__ mask, const OffT* __restrict__ off, int64_t n, Pair* sums) {
    __shared__ Pair s_warp[SC_NT / 32];
    const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_IPT;
    Pair t{0, 0};
#pragma unroll
    for (int k = 0; k < SC_IPT; ++k)
        if (base + k < n) {
            const Pair it = frontier_item(mask, off, base + k);
            t.a += it.a;
            t.b += it.b;
        }
    Pair tot;
    block_excl_scan2(t, s_warp, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(SC_NT) k_fscan_sums(Pair* sums, int64_t m) {
    __shared__ Pair s_warp[SC_NT / 32];
    Pair carry{0, 0};
    for (int64_t c = 0; c < m; c += SC_NT) {
        const int64_t i = c + threadIdx.x;
        const Pair v = i < m ? sums[i] : Pair{0, 0};
        Pair tot;
        const Pair ex = block_excl_scan2(v, s_warp, &tot);
        __syncthreads();
        if (i < m) sums[i] = Pair{carry.a + ex.a, carry.b + ex.b};
        carry.a += tot.a;
        carry.b += tot.b;
        __syncthreads();
    }
    if (threadIdx.x == 0) sums[m] = carry;
}

// active[slot] = v, fo[slot] = edge offset; fo[n_active] and count[0..1] = totals
template <class OffT>
__global__ void __launch_bounds__(SC_NT)
    k_fscan_down(const uint8_t* __restrict__ mask, const OffT* __restrict__ off, int64_t n,
                 const Pair* __restrict__ sums, int64_t nb, int32_t* __restrict__ active,
                 int64_t* __restrict__ fo, int64_t* __restrict__ count) {
    __shared__ Pair s_warp[SC_NT / 32];
    const int64_t base = (int64_t)blockIdx.x * SC_TILE + (int64_t)threadIdx.x * SC_IPT;
    Pair v[SC_IPT], t{0, 0};
#pragma unroll
    for (int k = 0; k < SC_IPT; ++k) {
        v[k] = base + k < n ? frontier_item(mask, off, base + k) : Pair{0, 0};
        t.a += v[k].a;
        t.b += v[k].b;
    }
    const Pair ex = block_excl_scan2(t, s_warp, nullptr);
    Pair run{sums[blockIdx.x].a + ex.a, sums[blockIdx.x].b + ex.b};
#pragma unroll
    for (int k = 0; k < SC_IPT; ++k) {
        if (v[k].a) {
            active[run.a] = (int32_t)(base + k);
            fo[run.a] = run.b;
        }
        run.a += v[k].a;
        run.b += v[k].b;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const Pair tot = sums[nb];
        fo[tot.a] = tot.b;
        count[0] = tot.a;
        count[1] = tot.b;
    }
}

// ---- relaxation ------------------------------------------------------------------------
struct SsspOp {
    double* dist;
    bool filter;   // read dist[v] before the atomic (work_oriented; see relax)
    __device__ __forceinline__ void prep(int64_t u, double& du) const { du = dist[u]; }
    template <class ValT>
    __device__ __forceinline__ bool relax(int64_t v, ValT w, double du) const {
        const double nd = du + (double)w;
        // dist only decreases, so a stale (L1) read is an upper bound: when it
        // already beats nd the atomic could not improve v and is skipped. Under
        // work_oriented this removes most atomics (C3-like R-MAT: 6.4 -> 4.5 ms);
        // the thread/group kernels walk long rows serially, where the extra
        // dependent load costs more than the atomics it saves (+9-23%).
        if (filter && !(nd < dist[v])) return false;
        const unsigned long long old =
            atomicMin(reinterpret_cast<unsigned long long*>(dist + v), (unsigned long long)__double_as_longlong(nd));
        return nd < __longlong_as_double((long long)old);
    }
};
struct BfsOp {
    int64_t* depth;
    int64_t next;
    __device__ __forceinline__ void prep(int64_t, double&) const {}
    template <class ValT>
    __device__ __forceinline__ bool relax(int64_t v, ValT, double) const {
        if (((volatile int64_t*)depth)[v] < 0) {
            depth[v] = next;
            return true;
        }
        return false;
    }
};

// Edges [e0, e1) of one source, four at a time: the column / weight loads and the
// four atomics are all issued before any result is used, so a thread keeps
// several relaxations in flight instead of one dependent round trip per edge.
template <class OffT, class ValT, class Op>
__device__ __forceinline__ void relax_edges(const Csr<OffT, ValT>& G, const Op& op, uint8_t* out,
                                            int64_t e0, int64_t e1, double du) {
    constexpr int R = 4;
    int64_t e = e0;
    for (; e + R <= e1; e += R) {
        int32_t v[R];
        ValT w[R];
        bool hit[R];
#pragma unroll
        for (int k = 0; k < R; ++k) { v[k] = __ldg(G.col + e + k); w[k] = __ldg(G.val + e + k); }
#pragma unroll
        for (int k = 0; k < R; ++k) hit[k] = op.relax(v[k], w[k], du);
#pragma unroll
        for (int k = 0; k < R; ++k)
            if (hit[k]) out[v[k]] = 1;
    }
    for (; e < e1; ++e) {
        const int64_t v = __ldg(G.col + e);
        const ValT w = __ldg(G.val + e);
        if (op.relax(v, w, du)) out[v] = 1;
    }
}

// thread_mapped: lane l owns frontier tiles l, l+P, ...
template <class OffT, class ValT, class Op>
__global__ void k_relax_thread(Csr<OffT, ValT> G, Op op, const int32_t* __restrict__ active,
                               int64_t n_active, int64_t lanes, uint8_t* __restrict__ out) {
    const int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= lanes) return;
    for (int64_t t = lane; t < n_active; t += lanes) {
        const int64_t u = active[t];
        double du = 0.0;
        op.prep(u, du);
        relax_edges(G, op, out, (int64_t)__ldg(G.off + u), (int64_t)__ldg(G.off + u + 1), du);
    }
}

// work_oriented: merge path over (frontier tiles, edges); fo = frontier offsets
template <class OffT, class ValT, class Op>
__global__ void k_relax_merge(Csr<OffT, ValT> G, Op op, const int32_t* __restrict__ active,
                              const int64_t* __restrict__ fo, int64_t n_active, int64_t lanes,
                              int64_t items, uint8_t* __restrict__ out) {
    const int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= lanes) return;
    const int64_t atoms = fo[n_active], total = n_active + atoms;
    auto search = [&](int64_t d) {   // greatest t with fo[t] <= d - t
        int64_t lo = max((int64_t)0, d - atoms), hi = min(d, n_active);
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (fo[mid] <= d - mid) lo = mid;
            else hi = mid - 1;
        }
        return lo;
    };
    const int64_t d0 = min(lane * items, total), d1 = min((lane + 1) * items, total);
    const int64_t t0 = search(d0), t1 = search(d1);
    int64_t a = d0 - t0;
    const int64_t a1 = d1 - t1;
    // tile portions of the slice, as _walk_merge_path_atoms hands them out
    for (int64_t t = t0; t <= t1 && t < n_active; ++t) {
        const int64_t end = t < t1 ? fo[t + 1] : a1;
        if (a < end) {
            const int64_t u = active[t];
            double du = 0.0;
            op.prep(u, du);
            const int64_t shift = (int64_t)__ldg(G.off + u) - fo[t];
            relax_edges(G, op, out, shift + a, shift + end, du);
            a = end;
        }
    }
}

// group_mapped: groups own blocks of tpb frontier tiles, members stride atoms;
// get_tile by monotone advance over fo (executor.py:149-168)
template <class OffT, class ValT, class Op>
__global__ void k_relax_group(Csr<OffT, ValT> G, Op op, const int32_t* __restrict__ active,
                              const int64_t* __restrict__ fo, int64_t n_active, int64_t lanes,
                              int64_t gs, int64_t tpb, uint8_t* __restrict__ out) {
    const int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= lanes) return;
    const int64_t groups = (lanes + gs - 1) / gs;
    const int64_t g = lane / gs, m = lane - g * gs;
    const int64_t members = min(gs, lanes - g * gs);
    const int64_t blocks = (n_active + tpb - 1) / tpb;
    for (int64_t b = g; b < blocks; b += groups) {
        const int64_t tb = b * tpb, tc = min(tpb, n_active - tb);
        const int64_t base = fo[tb], tot = fo[tb + tc] - base;
        int64_t t = tb;
        constexpr int R = 4;   // four member-stride atoms per round, relaxations in flight together
        for (int64_t k0 = m; k0 < tot; k0 += R * members) {
            int32_t v[R];
            ValT w[R];
            double du[R];
            bool live[R], hit[R];
#pragma unroll
            for (int q = 0; q < R; ++q) {
                const int64_t a = base + k0 + q * members;
                live[q] = k0 + q * members < tot;
                v[q] = 0;
                w[q] = (ValT)0;
                du[q] = 0.0;
                if (live[q]) {
                    while (fo[t + 1] <= a) ++t;   // get_tile by monotone advance
                    const int64_t u = active[t];
                    op.prep(u, du[q]);
                    const int64_t e = (int64_t)__ldg(G.off + u) + (a - fo[t]);
                    v[q] = __ldg(G.col + e);
                    w[q] = __ldg(G.val + e);
                }
            }
#pragma unroll
            for (int q = 0; q < R; ++q) hit[q] = live[q] && op.relax(v[q], w[q], du[q]);
#pragma unroll
            for (int q = 0; q < R; ++q)
                if (hit[q]) out[v[q]] = 1;
        }
    }
}

__global__ void k_init_sssp(double* dist, uint8_t* mask, int64_t n, int64_t src) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    dist[i] = i == src ? 0.0 : __longlong_as_double(0x7ff0000000000000LL);
    mask[i] = i == src;
}
__global__ void k_init_bfs(int64_t* depth, uint8_t* mask, int64_t n, int64_t src) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    depth[i] = i == src ? 0 : -1;
    mask[i] = i == src;
}

// ---- host side -------------------------------------------------------------------------
struct FrontierWs {
    uint8_t* mask_in;
    uint8_t* mask_out;
    int32_t* active;
    int64_t* fo;
    int64_t* sums;
    int64_t* count;   // [2]: active count, scratch
};

static size_t up256(size_t b) { return (b + 255) / 256 * 256; }

size_t frontier_workspace(int64_t n) {
    const size_t nb = (size_t)scan_blocks(n) + 1;
    return up256((size_t)n) * 2 + up256((size_t)n * 4) + up256((size_t)(n + 1) * 8) + up256(nb * 16) +
           up256(16);
}

static FrontierWs carve(void* ws, int64_t n) {
    unsigned char* p = (unsigned char*)ws;
    FrontierWs w{};
    w.mask_in = p; p += up256((size_t)n);
    w.mask_out = p; p += up256((size_t)n);
    w.active = (int32_t*)p; p += up256((size_t)n * 4);
    w.fo = (int64_t*)p; p += up256((size_t)(n + 1) * 8);
    w.sums = (int64_t*)p; p += up256(((size_t)scan_blocks(n) + 1) * 16);
    w.count = (int64_t*)p;
    return w;
}

int frontier_compact(const uint8_t* mask, int64_t n, int32_t* active, int64_t* count_dev, void* ws,
                     cudaStream_t s) {
    FrontierWs w = carve(ws, n);
    return scan_run<FlagOf, true>(FlagOf{mask}, n, w.sums, nullptr, active, count_dev, s);
}

static int64_t frontier_lanes(int schedule, int64_t n_active, int64_t atoms, int64_t lanes,
                              int64_t gs, int64_t tpb) {
    if (lanes > 0) return lanes;
    switch (schedule) {
        case LW_THREAD_MAPPED: {
            const int64_t cap = (int64_t)sm_count() * 2048;
            return n_active < cap ? (n_active > 0 ? n_active : 1) : cap;
        }
        case LW_MERGE_PATH: return (n_active + atoms) > 0 ? ceil_div(n_active + atoms, 16) : 1;
        default: return group_auto_lanes(n_active, gs, tpb);
    }
}

template <class OffT, class ValT, class Op>
static int relax_typed(const lw_csr_t* H, const Op& op, const int32_t* active, int64_t n_active,
                       const int64_t* fo, int64_t atoms, uint8_t* out, int schedule, int64_t lanes,
                       int64_t gs, int64_t tpb, cudaStream_t s) {
    Csr<OffT, ValT> G{H->rows, H->cols, H->nnz, (const OffT*)H->row_offsets, H->col_indices,
                      (const ValT*)H->values};
    const int64_t P = frontier_lanes(schedule, n_active, atoms, lanes, gs, tpb);
    const unsigned grid = (unsigned)ceil_div(P, 256);
    switch (schedule) {
        case LW_THREAD_MAPPED:
            k_relax_thread<OffT, ValT, Op><<<grid, 256, 0, s>>>(G, op, active, n_active, P, out);
            break;
        case LW_MERGE_PATH: {
            const int64_t total = n_active + atoms;
            const int64_t items = total > 0 ? ceil_div(total, P) : 0;
            k_relax_merge<OffT, ValT, Op><<<grid, 256, 0, s>>>(G, op, active, fo, n_active, P, items, out);
            break;
        }
        case LW_GROUP_MAPPED:
            k_relax_group<OffT, ValT, Op><<<grid, 256, 0, s>>>(G, op, active, fo, n_active, P, gs, tpb, out);
            break;
        default: return LW_E_INVALID_ARG;
    }
    LW_LAUNCH_CHECK();
    return LW_OK;
}

template <class Op>
static int relax_dispatch(const lw_csr_t* H, const Op& op, const int32_t* active, int64_t n_active,
                          const int64_t* fo, int64_t atoms, uint8_t* out, int schedule,
                          int64_t lanes, int64_t gs, int64_t tpb, cudaStream_t s) {
    const bool o32 = H->offset_bits == 32;
    if (H->dtype == LW_F32)
        return o32 ? relax_typed<int32_t, float>(H, op, active, n_active, fo, atoms, out, schedule, lanes, gs, tpb, s)
                   : relax_typed<int64_t, float>(H, op, active, n_active, fo, atoms, out, schedule, lanes, gs, tpb, s);
    return o32 ? relax_typed<int32_t, double>(H, op, active, n_active, fo, atoms, out, schedule, lanes, gs, tpb, s)
               : relax_typed<int64_t, double>(H, op, active, n_active, fo, atoms, out, schedule, lanes, gs, tpb, s);
}

// One pass over an already compacted frontier (active[n_active], host count):
// computes the frontier offsets, zeroes out_frontier, relaxes.
template <class Op>
static int frontier_pass(const lw_csr_t* H, const Op& op, const int32_t* active, int64_t n_active,
                         uint8_t* out, int schedule, int64_t lanes, int64_t gs, int64_t tpb,
                         void* ws, cudaStream_t s) {
    FrontierWs w = carve(ws, H->rows);
    LW_TRY(cudaMemsetAsync(out, 0, (size_t)H->rows, s));
    if (n_active == 0) return LW_OK;
    int64_t atoms = 0;
    if (schedule != LW_THREAD_MAPPED) {
        int rc = scan_run<DegreeOf, false>(DegreeOf{H->row_offsets, H->offset_bits, active}, n_active,
                                           w.sums, w.fo, nullptr, nullptr, s);
        if (rc) return rc;
        LW_TRY(cudaMemcpyAsync(&atoms, w.fo + n_active, 8, cudaMemcpyDeviceToHost, s));
        LW_TRY(cudaStreamSynchronize(s));
    }
    return relax_dispatch(H, op, active, n_active, w.fo, atoms, out, schedule, lanes, gs, tpb, s);
}

int sssp_pass(const lw_csr_t* H, const int32_t* active, int64_t n_active, double* dist,
              uint8_t* out, int schedule, int64_t lanes, int64_t gs, int64_t tpb, void* ws,
              cudaStream_t s) {
    return frontier_pass(H, SsspOp{dist, schedule == LW_MERGE_PATH}, active, n_active, out, schedule, lanes, gs, tpb, ws, s);
}

int bfs_pass(const lw_csr_t* H, const int32_t* active, int64_t n_active, int64_t* depth,
             int64_t next, uint8_t* out, int schedule, int64_t lanes, int64_t gs, int64_t tpb,
             void* ws, cudaStream_t s) {
    return frontier_pass(H, BfsOp{depth, next}, active, n_active, out, schedule, lanes, gs, tpb, ws, s);
}

// Whole traversal: loop passes until the frontier is empty (one host sync per pass
// for the frontier size, as the reference's `while in_frontier.any()`).
template <bool SSSP>
static int traverse(const lw_csr_t* H, int64_t src, void* result, int schedule, int64_t lanes,
                    int64_t gs, int64_t tpb, void* ws, int64_t* passes, cudaStream_t s) {
    const int64_t n = H->rows;
    FrontierWs w = carve(ws, n);
    const unsigned g = (unsigned)ceil_div(n, 256);
    if (SSSP) k_init_sssp<<<g, 256, 0, s>>>((double*)result, w.mask_in, n, src);
    else k_init_bfs<<<g, 256, 0, s>>>((int64_t*)result, w.mask_in, n, src);
    LW_LAUNCH_CHECK();
    int64_t level = 0, np = 0;
    uint8_t* in = w.mask_in;
    uint8_t* out = w.mask_out;
    const int64_t nb = scan_blocks(n);
    Pair* sums = (Pair*)w.sums;
    // pinned (n_active, atoms) read back once per pass: one 16-byte buffer per host
    // thread, allocated on first use and kept (cudaFreeHost would synchronize the
    // whole device on every call); a call completes before it returns, so the
    // calls of one thread never share it concurrently
    static thread_local int64_t* hc = nullptr;
    if (!hc) LW_TRY(cudaHostAlloc((void**)&hc, 16, cudaHostAllocPortable));
    int rc = LW_OK;
    for (;;) {
        // one sweep: active[] = flatnonzero(in), fo[] = frontier edge offsets
        if (H->offset_bits == 32) {
            const int32_t* o = (const int32_t*)H->row_offsets;
            k_fscan_up<int32_t><<<(unsigned)nb, SC_NT, 0, s>>>(in, o, n, sums);
            k_fscan_sums<<<1, SC_NT, 0, s>>>(sums, nb);
            k_fscan_down<int32_t><<<(unsigned)nb, SC_NT, 0, s>>>(in, o, n, sums, nb, w.active, w.fo, w.count);
        } else {
            const int64_t* o = (const int64_t*)H->row_offsets;
            k_fscan_up<int64_t><<<(unsigned)nb, SC_NT, 0, s>>>(in, o, n, sums);
            k_fscan_sums<<<1, SC_NT, 0, s>>>(sums, nb);
            k_fscan_down<int64_t><<<(unsigned)nb, SC_NT, 0, s>>>(in, o, n, sums, nb, w.active, w.fo, w.count);
        }
        if ((rc = (int)cudaGetLastError())) break;
        if ((rc = (int)cudaMemcpyAsync(hc, w.count, 16, cudaMemcpyDeviceToHost, s))) break;
        if ((rc = (int)cudaStreamSynchronize(s))) break;
        const int64_t n_active = hc[0], atoms = hc[1];
        if (n_active == 0) break;
        if ((rc = (int)cudaMemsetAsync(out, 0, (size_t)n, s))) break;
        rc = SSSP ? relax_dispatch(H, SsspOp{(double*)result, schedule == LW_MERGE_PATH}, w.active, n_active, w.fo, atoms, out,
                                   schedule, lanes, gs, tpb, s)
                  : relax_dispatch(H, BfsOp{(int64_t*)result, level + 1}, w.active, n_active, w.fo, atoms,
                                   out, schedule, lanes, gs, tpb, s);
        if (rc) break;
        uint8_t* t = in;
        in = out;
        out = t;
        ++level;
        ++np;
    }
    if (rc) return rc;
    if (passes) *passes = np;
    return LW_OK;
}

int sssp_run(const lw_csr_t* H, int64_t src, double* dist, int schedule, int64_t lanes, int64_t gs,
             int64_t tpb, void* ws, int64_t* passes, cudaStream_t s) {
    return traverse<true>(H, src, dist, schedule, lanes, gs, tpb, ws, passes, s);
}
int bfs_run(const lw_csr_t* H, int64_t src, int64_t* depth, int schedule, int64_t lanes, int64_t gs,
            int64_t tpb, void* ws, int64_t* passes, cudaStream_t s) {
    return traverse<false>(H, src, depth, schedule, lanes, gs, tpb, ws, passes, s);
}

}  // namespace lw
