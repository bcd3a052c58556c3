// spmv_group_mapped.cu — group_mapped schedule (warp tiles, block tiles, general groups).
//
// Schedule (reference schedules.py:137-167, executor.py:149-168):
// lanes are cut into groups of group_size (the last group may be short,
// executor.py:65-72); tile blocks of tiles_per_block tiles are dealt to groups in
// group-stride order (block b -> group b mod G); inside a block, member m of a
// group with `members` lanes takes block-local atoms m, m+members, ... and each
// atom is attributed to the tile whose exclusive-prefix interval contains it
// (get_tile, schedules.py:162-167). Lanes are device threads, so the per-lane atom
// multisets equal executor.imbalance()/execute_tile_major for the same P.
//
// Kernels (replace _fast.spmv_group_mapped, _fast.py:55-77):
//  * k_group_warp   (group_size = tiles_per_block = 32): a warp is a group. The
//    block plan is a warp-shuffle exclusive scan of the 32 per-tile atom counts;
//    atom -> tile (get_tile) follows the tile starts that fall inside each 32-atom
//    step (a ballot over the plan, one shuffle per start); each step is reduced
//    with a ballot-driven shuffle segmented reduction and the run heads add into a
//    per-warp shared accumulator, so y is written once per tile, coalesced, with
//    a fixed summation order.
//  * k_group_block<NT> (group_size = tiles_per_block = NT in {64,128,256}): the
//    CTA is a group; the plan is a block-wide scan into shared memory, atom ->
//    tile is a log2(NT)-probe search in shared memory, per-warp shared
//    accumulators (combined in warp order) keep the result deterministic.
//  * any other group_size / tiles_per_block / lane count: k_group_tiles, one
//    thread per tile summing the tile's atoms in the reference's member-major
//    order (bit-identical to the reference's fp64 y, deterministic); probe runs
//    first execute k_group_generic — one thread per lane running the reference's
//    member loop with a monotone tile advance (_fast.py:75-76) — to record the
//    lane -> atom -> tile assignment.
#include <algorithm>
#include <climits>
#include <type_traits>

#include "lw_common.cuh"

namespace lw {

#ifndef LW_GU
#define LW_GU 4
#endif
constexpr int GU = LW_GU;     // member-stride steps whose loads are in flight together
constexpr int GU_LONG = 64;  // blocks with >= GU_LONG*group atoms use the GU-step loop

// Products of the atoms a member takes in GU consecutive member-stride steps
// (local atoms k0 + u*STRIDE + m): every col/val load first, then every gather.
template <class ValT, int U, int STRIDE, class OffT>
__device__ __forceinline__ void gather_steps(const Csr<OffT, ValT>& A, const ValT* __restrict__ x,
                                             int64_t base, OffT k0, int m, OffT total,
                                             double (&p)[U]) {
    int32_t c[U];
    ValT v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const OffT k = k0 + u * STRIDE + m;
        const bool valid = k < total;
        c[u] = valid ? ld_stream(A.col + base + k) : 0;
        v[u] = valid ? ld_stream(A.val + base + k) : (ValT)0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const bool valid = k0 + u * STRIDE + m < total;
        p[u] = valid ? (double)v[u] * (double)ld_gather(x + c[u]) : 0.0;
    }
}

// The same U steps split in two, for the software-pipelined long-block loop: the
// next U steps' col/val stream in while this U steps' gathers are in flight.
template <class ValT, int U>
struct StepLoads {
    int32_t c[U];
    ValT v[U];
};
template <class ValT, int U, int STRIDE, class OffT>
__device__ __forceinline__ void load_steps(const Csr<OffT, ValT>& A, int64_t base, OffT k0, int m,
                                           OffT total, StepLoads<ValT, U>& L) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const OffT k = k0 + u * STRIDE + m;
        const bool valid = k < total;
        L.c[u] = valid ? ld_stream(A.col + base + k) : 0;
        L.v[u] = valid ? ld_stream(A.val + base + k) : (ValT)0;
    }
}
template <class ValT, int U, int STRIDE, class OffT>
__device__ __forceinline__ void gather_loaded(const StepLoads<ValT, U>& L, const ValT* __restrict__ x,
                                              OffT k0, int m, OffT total, double (&p)[U]) {
    // every gather issued before the first product: written as one expression
    // per step, ptxas placed each product right after its gather and the warp
    // waited out U round trips per iteration (C3 fp32 11.9 -> 10.2 ms, power-law
    // skew 1.05 3.87 -> 2.85 ms with the split)
    ValT g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) g[u] = k0 + u * STRIDE + m < total ? ld_gather(x + L.c[u]) : (ValT)0;
#pragma unroll
    for (int u = 0; u < U; ++u) p[u] = (double)L.v[u] * (double)g[u];
}

// Cooperative-path iterations whose atoms all fall in one tile (the inside of a
// long row): each lane adds its products to a running fp64 sum, and the warp
// reduces it (fixed xor-butterfly order) into the tile's accumulator once, when
// the run of single-tile iterations ends. Warp-uniform state.
// Block tiles: 1 = one block-uniform get_tile(k0) per iteration decides (C3 fp32 /
// fp64 8.37 / 9.90 -> 5.36 / 7.06 ms, power-law skew 1.05 1.21 / 1.40 -> 0.66 /
// 0.87; C1 +6% / +13%: ~10 rows per iteration never qualify); 2 = a warp vote
// over the per-atom searches it already does (C3 8.03 ms: the searches are the
// cost); 0 = off. Gating the check on a block-wide "has a row >= GU*NT atoms"
// flag cost the loop its register allocation (C3 6.82 ms).
#ifndef LW_G_SINGLE
#define LW_G_SINGLE 1
#endif
#ifndef LW_GW_SINGLE    // warp tiles: fp32 power-law -15% but fp64 C3 11.4 -> 17.2 ms and C2b
#define LW_GW_SINGLE 0  // +12% (63 registers, fewer resident groups), off
#endif
struct SingleTileRun {
    double sum = 0.0;
    int tile = -1;
    template <int U>
    __device__ __forceinline__ void take(int t, const double (&p)[U], int lane, double* acc) {
        if (t != tile) { flush(lane, acc); tile = t; }
#pragma unroll
        for (int u = 0; u < U; ++u) sum += p[u];
    }
    __device__ __forceinline__ void flush(int lane, double* acc) {
        if (tile < 0) return;
        double r = sum;
#pragma unroll
        for (int d = kWarp / 2; d >= 1; d >>= 1) r += __shfl_xor_sync(0xffffffffu, r, d);
        if (lane == 0) acc[tile] += r;
        __syncwarp();
        sum = 0.0;
        tile = -1;
    }
};

// ---- warp tiles -------------------------------------------------------------------
#ifndef LW_GW_CAP      // atoms per warp block staged in shared memory (0 = off)
#define LW_GW_CAP 576
#endif
#ifndef LW_GW_SU       // member-stride steps in flight on the staged path
#define LW_GW_SU 2
#endif
constexpr int GW_SU = LW_GW_SU;
#ifndef LW_GW_LONG     // longest row the staged path sums in one lane
#define LW_GW_LONG 128
#endif
constexpr int GW_LONG = LW_GW_LONG;
#ifndef LW_GW_MINB
#define LW_GW_MINB 0
#endif
// The staged-block path of k_group_warp (see the kernel).
template <class OffT, class ValT, int CAP>
__device__ __forceinline__ void group_warp_staged(const Csr<OffT, ValT>& A, const ValT* __restrict__ x,
                                               ValT* __restrict__ y, int64_t tb, int tc, int64_t base,
                                               OffT excl, OffT incl, OffT cnt, ValT* sp) {
    const int lane = threadIdx.x & (kWarp - 1);
    int ta = 0;
    while (ta < tc) {
        const OffT sa = shfl(excl, ta);
        // tiles ta .. te-1 whose atoms end within sa + CAP (incl is increasing)
        const unsigned fit = __ballot_sync(0xffffffffu, lane >= ta && lane < tc && incl - sa <= (OffT)CAP);
        const int te = 32 - __clz(fit);
        const OffT sb = shfl(incl, te - 1);
        for (OffT k0 = sa & ~(OffT)(kWarp - 1); k0 < sb; k0 += GW_SU * kWarp) {
            int32_t c[GW_SU];
            ValT v[GW_SU];
#pragma unroll
            for (int u = 0; u < GW_SU; ++u) {
                const OffT k = k0 + u * kWarp + lane;
                const bool valid = k >= sa && k < sb;
                c[u] = valid ? ld_stream(A.col + base + k) : 0;
                v[u] = valid ? ld_stream(A.val + base + k) : (ValT)0;
            }
#pragma unroll
            for (int u = 0; u < GW_SU; ++u) {
                const OffT k = k0 + u * kWarp + lane;
                if (k >= sa && k < sb) sp[k - sa] = v[u] * ld_gather(x + c[u]);
            }
        }
        __syncwarp();
        if (lane >= ta && lane < te) {
            double acc = 0.0;
            const int e0 = (int)(excl - sa), n = (int)cnt;
            for (int j = 0; j < n; ++j) acc += (double)sp[e0 + j];
            y[tb + lane] = (ValT)acc;
        }
        __syncwarp();
        ta = te;
    }
}

// The cooperative path of k_group_warp (blocks with long rows, and every block of
// the instrumented variant).
template <class OffT, class ValT, bool PROBE>
__device__ __forceinline__ void group_warp_coop(const Csr<OffT, ValT>& A, const ValT* __restrict__ x,
                                             ValT* __restrict__ y, const Probe& probe, int64_t tb,
                                             int tc, int64_t base, OffT cnt, OffT excl, OffT total,
                                             int64_t glane, int64_t& mine, double* acc) {
    const int lane = threadIdx.x & (kWarp - 1);
    acc[lane] = 0.0;
    __syncwarp();
    // U member-stride steps per iteration (lane takes local atoms k0+u*32+lane),
    // all their loads and gathers in flight before the first reduction; U = GU
    // only for long blocks (short ones would waste the padded steps)
    int t_cur = 0;   // tile of the previous step's last atom (warp-uniform)
    auto steps = [&](auto uc) {
      constexpr int U = decltype(uc)::value;
      StepLoads<ValT, U> cur, nxt;
      if (U > 1) load_steps<ValT, U, kWarp>(A, base, (OffT)0, lane, total, cur);
      SingleTileRun run;
      for (OffT k0 = 0; k0 < total; k0 += U * kWarp) {
        double p[U];
        if (U > 1) {   // long block: next steps' loads overlap these gathers
            load_steps<ValT, U, kWarp>(A, base, (OffT)(k0 + U * kWarp), lane, total, nxt);
            gather_loaded<ValT, U, kWarp>(cur, x, k0, lane, total, p);
            cur = nxt;
          if (LW_GW_SINGLE) {
            // every atom of the iteration in one tile (inside a long row): no
            // get_tile search and no segmented reductions, the products go to a
            // per-lane running sum that is reduced once when the run of such
            // iterations ends (deterministic order)
            // get_tile(k0): the largest tile starting at or before k0 (one ballot)
            const int t0 = 31 - __clz(__ballot_sync(0xffffffffu, lane < tc && excl <= k0));
            const OffT last = k0 + (OffT)(U * kWarp) < total ? k0 + (OffT)(U * kWarp) : total;
            if (shfl((OffT)(excl + cnt), t0) >= last) {
                run.take<U>(t0, p, lane, acc);
                if (PROBE) {
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (k0 + u * kWarp + lane < total) { probe_atom(probe, base + k0 + u * kWarp + lane, glane, tb + t0); ++mine; }
                }
                continue;
            }
            run.flush(lane, acc);
          }
        } else {
            gather_steps<ValT, U, kWarp>(A, x, base, k0, lane, total, p);
        }
        // non-empty tiles starting inside this step's atoms (lane j <-> tile j)
        const uint32_t starts = U == 1 ? __ballot_sync(
            0xffffffffu, lane < tc && cnt > 0 && excl >= k0 && excl < k0 + (OffT)kWarp) : 0u;
        const int t_it = t_cur;
        int t_next = t_cur;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const OffT k = k0 + u * kWarp + lane;
            const bool valid = k < total;
            // get_tile (largest non-empty t with excl[t] <= k): the step's atoms
            // are consecutive, so only the non-empty tiles that START inside the
            // step can change the tile; lane j flags tile j, and the few flagged
            // starts are broadcast in order (one shuffle each, none inside a
            // long row) instead of a 5-probe search per atom
            // (long blocks, U > 1, keep the independent 5-probe search: there the
            // steps' searches overlap, and R-MAT / power-law blocks measured 15-25%
            // slower with the start-following loop)
            int t = 0;
            if (U == 1) {
                t = t_it;
                for (uint32_t sm = starts; sm; sm &= sm - 1) {
                    const int j = __ffs(sm) - 1;
                    if (k >= shfl(excl, j)) t = j;
                }
                t_next = shfl(t, kWarp - 1);
            } else {
#pragma unroll
                for (int s = kWarp / 2; s >= 1; s >>= 1) {
                    const OffT e = shfl(excl, t + s);
                    if (t + s < tc && e <= k) t += s;
                }
            }
            if (PROBE && valid) { probe_atom(probe, base + k, glane, tb + t); ++mine; }
            const int key = valid ? t : INT_MAX;
            const int prev = shfl_up(key, 1);
            const bool head = lane == 0 || prev != key;
            const uint32_t heads = __ballot_sync(0xffffffffu, head);
            // a step's partial sums (<= 32 products) in the value precision
            const double sum = (double)warp_segsum_heads<ValT>((ValT)p[u], lane, heads);
            if (valid && head) acc[t] += sum;
            __syncwarp();
        }
        t_cur = t_next;
      }
      run.flush(lane, acc);
    };
    if (total >= (OffT)(GU_LONG * kWarp)) steps(std::integral_constant<int, GU>{});
    else steps(std::integral_constant<int, 1>{});
    if (lane < tc) y[tb + lane] = (ValT)acc[lane];
    __syncwarp();
}

// MODE: GW_ALL runs every block through the cooperative path (the instrumented
// variant); the uninstrumented SpMV is two launches over the same groups and
// blocks, GW_STAGED (blocks whose rows are all <= GW_LONG atoms, staged) then
// GW_COOP (the other blocks, cooperative). Each block is computed by one of them
// in full, so y does not depend on which warp ran it; the two paths are separate
// kernels because inlined together they cost the cooperative loop its register
// allocation (C3 12.1 -> 17.3 ms, and 24 ms as a non-inlined call).
constexpr int GW_ALL = 0, GW_STAGED = 1, GW_COOP = 2;
template <class OffT, class ValT, bool PROBE, int MODE = GW_ALL>
__global__ void __launch_bounds__(256, LW_GW_MINB)
    k_group_warp(Csr<OffT, ValT> A, const ValT* __restrict__ x, ValT* __restrict__ y,
                 int64_t groups, Probe probe) {
    __shared__ double s_acc[8][kWarp];
    const int lane = threadIdx.x & (kWarp - 1), warp = threadIdx.x >> 5;
    const int64_t g = (int64_t)blockIdx.x * 8 + warp;
    if (g >= groups) return;
    const int64_t nblocks = (A.rows + kWarp - 1) / kWarp;
    const int64_t glane = g * kWarp + lane;
    int64_t mine = 0;
    for (int64_t b = g; b < nblocks; b += groups) {
        const int64_t tb = b * kWarp;
        const int tc = (int)min((int64_t)kWarp, A.rows - tb);
        // per-tile atom counts -> warp exclusive prefix sum (the group plan)
        const OffT lo_off = lane < tc ? A.off[tb + lane] : (OffT)0;
        const OffT hi_off = lane < tc ? A.off[tb + lane + 1] : (OffT)0;
        const OffT cnt = hi_off - lo_off;
        OffT incl = cnt;
#pragma unroll
        for (int d = 1; d < kWarp; d <<= 1) {
            const OffT o = shfl_up(incl, d);
            if (lane >= d) incl += o;
        }
        const OffT excl = incl - cnt;
        const OffT total = shfl(incl, kWarp - 1);
        const int64_t base = (int64_t)shfl(lo_off, 0);
        if constexpr (MODE != GW_ALL) {
            // Staged block (rows up to GW_LONG atoms): the members compute their
            // atoms' products exactly as the schedule assigns them (member m: local
            // atoms m, m+32, ..., GW_SU steps of loads in flight) into shared memory,
            // one tile-aligned segment of <= CAP atoms at a time, and the lane owning
            // tile t then sums the tile's products in atom order (fp64). No per-atom
            // get_tile and no per-step segmented reduction; integer data stays
            // bit-exact (same products, exact fp64 sums). Blocks with a longer row
            // take the cooperative path (one lane would serialise the row).
            constexpr int CAP = LW_GW_CAP > 0 ? LW_GW_CAP * 4 / (int)sizeof(ValT) : 1;
            OffT mx = cnt;
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) {
                const OffT o = __shfl_xor_sync(0xffffffffu, mx, d);
                mx = o > mx ? o : mx;
            }
            const bool staged = mx <= (OffT)(GW_LONG < CAP ? GW_LONG : CAP);
            if constexpr (MODE == GW_STAGED) {
                if (staged) {
                    __shared__ ValT s_prod[8][CAP];
                    group_warp_staged<OffT, ValT, CAP>(A, x, y, tb, tc, base, excl, incl, cnt,
                                                       s_prod[warp]);
                }
                continue;
            } else {
                if (staged) continue;
            }
        }
        group_warp_coop<OffT, ValT, PROBE>(A, x, y, probe, tb, tc, base, cnt, excl, total, glane, mine,
                                           s_acc[warp]);
    }
    if (PROBE && probe.lane_atoms) probe.lane_atoms[glane] = mine;
}

// ---- block tiles ------------------------------------------------------------------
// Block selection of the uninstrumented block-tile SpMV: a block is STAGED when
// all its rows have <= GB_LONG atoms and either none exceeds GB_LONG/4 or at
// least a quarter do (no lone long row for one thread to sum while the CTA
// waits at the barrier); the other blocks run the cooperative path. Unlike the
// warp tiles (two launches), both paths live in one kernel and share one
// shared-memory buffer: as two launches the staged launch's time adds to the
// cooperative launch's tail on power-law inputs (C4 skew 1.05 fp32 1.22 ->
// 1.57 ms), in one grid the short blocks fill in under the long ones.
#ifndef LW_GB_LONG
#define LW_GB_LONG 64
#endif
#ifndef LW_GB_CAP      // atoms per staged segment (fp32 products; fp64 holds half)
#define LW_GB_CAP 4096
#endif
#ifndef LW_GB_SU       // member-stride steps of loads in flight on the staged path
#define LW_GB_SU 4
#endif
constexpr int GB_LONG = LW_GB_LONG, GB_SU = LW_GB_SU;
constexpr int GB_ALL = 0, GB_FUSED = 1;

template <class OffT>
__device__ __forceinline__ bool gb_staged_block(OffT cnt, int tc, int NT_) {
    // block max and sum of the row lengths (every thread of the CTA calls this)
    const bool too_long = __syncthreads_or(cnt > (OffT)GB_LONG);
    if (too_long) return false;
    const int n_ge = __syncthreads_count(cnt * 4 > (OffT)GB_LONG);   // rows above a quarter of the limit
    (void)NT_;
    // mostly-short blocks with a few long rows would serialise on those rows
    return n_ge == 0 || n_ge * 4 >= tc || tc < 8;
}

// Resident 256-thread CTAs the fused kernel's registers must allow (scaled by
// 256/NT): 6 -> 40 registers, no spills, 75% occupancy instead of 50% at 64.
// Block tile, fp32 / fp64: C2b 0.105 -> 0.077 / 0.151 -> 0.100 ms, C2u 0.182 ->
// 0.170 / 0.214 -> 0.182, C3 11.6 -> 8.4 / 13.1 -> 9.9 ms; power-law fp64 at
// skew <= 1.2 +1-3%. (5 -> 48 registers: C2b 0.087; 8 -> 32 registers spills.)
#ifndef LW_GB_MINB
#define LW_GB_MINB 6
#endif
template <class OffT, class ValT, int NT, bool PROBE, int MODE = GB_ALL>
__global__ void __launch_bounds__(NT, MODE == GB_FUSED ? LW_GB_MINB * 256 / NT : 1)
    k_group_block(Csr<OffT, ValT> A, const ValT* __restrict__ x, ValT* __restrict__ y,
                  int64_t groups, Probe probe) {
    constexpr int NW = NT / kWarp;
    constexpr int CAP = (MODE == GB_FUSED && LW_GB_CAP > 0) ? LW_GB_CAP * 4 / (int)sizeof(ValT) : 1;
    constexpr size_t RAW = sizeof(double) * NW * NT > sizeof(ValT) * CAP ? sizeof(double) * NW * NT
                                                                          : sizeof(ValT) * CAP;
    __shared__ OffT s_excl[NT + 1];
    __shared__ OffT s_wsum[NW];
    __shared__ __align__(16) unsigned char s_raw[RAW];   // cooperative accumulators | staged products
    double(*s_acc)[NT] = reinterpret_cast<double(*)[NT]>(s_raw);
    ValT* s_prod = reinterpret_cast<ValT*>(s_raw);
    const int tid = threadIdx.x, lane = tid & (kWarp - 1), warp = tid >> 5;
    const int64_t nblocks = (A.rows + NT - 1) / NT;
    const int64_t glane = (int64_t)blockIdx.x * NT + tid;
    int64_t mine = 0;
    for (int64_t b = blockIdx.x; b < nblocks; b += groups) {
        const int64_t tb = b * NT;
        const int tc = (int)min((int64_t)NT, A.rows - tb);
        const OffT cnt = tid < tc ? A.off[tb + tid + 1] - A.off[tb + tid] : (OffT)0;
        bool staged = false;
        if constexpr (MODE == GB_FUSED) staged = gb_staged_block<OffT>(cnt, tc, NT);
        if (staged) {
            // Staged block: the members compute their atoms' products exactly as
            // the schedule assigns them (member m: block-local atoms m, m+NT, ...;
            // GB_SU steps of loads in flight) into shared memory, one tile-aligned
            // segment of <= CAP atoms at a time; the thread owning tile t then sums
            // the tile's products in atom order (fp64) and writes y once. No per-atom
            // get_tile search, no per-step segmented reduction.
            OffT incl = cnt;
#pragma unroll
            for (int d = 1; d < kWarp; d <<= 1) {
                const OffT o = shfl_up(incl, d);
                if (lane >= d) incl += o;
            }
            if (lane == kWarp - 1) s_wsum[warp] = incl;
            __syncthreads();
            OffT wpre = 0;
            for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
            incl += wpre;
            const OffT excl = incl - cnt;
            s_excl[tid] = excl;
            if (tid == NT - 1) s_excl[NT] = incl;
            const int64_t base = (int64_t)A.off[tb];
            __syncthreads();
            int ta = 0;
            while (ta < tc) {
                const OffT sa = s_excl[ta];
                // tiles ta .. te-1 whose atoms end within sa + CAP (incl increases)
                const int te = ta + __syncthreads_count(tid >= ta && tid < tc && incl - sa <= (OffT)CAP);
                const OffT sb = s_excl[te];
                for (OffT k0 = sa - sa % (OffT)NT; k0 < sb; k0 += GB_SU * NT) {
                    int32_t c[GB_SU];
                    ValT v[GB_SU];
#pragma unroll
                    for (int u = 0; u < GB_SU; ++u) {
                        const OffT k = k0 + u * NT + tid;
                        const bool valid = k >= sa && k < sb;
                        c[u] = valid ? ld_stream(A.col + base + k) : 0;
                        v[u] = valid ? ld_stream(A.val + base + k) : (ValT)0;
                    }
#pragma unroll
                    for (int u = 0; u < GB_SU; ++u) {
                        const OffT k = k0 + u * NT + tid;
                        if (k >= sa && k < sb) s_prod[k - sa] = v[u] * ld_gather(x + c[u]);
                    }
                }
                __syncthreads();
                if (tid >= ta && tid < te) {
                    double acc = 0.0;
                    const int e0 = (int)(excl - sa), n = (int)cnt;
                    for (int j = 0; j < n; ++j) acc += (double)s_prod[e0 + j];
                    y[tb + tid] = (ValT)acc;
                }
                __syncthreads();
                ta = te;
            }
            continue;
        }
        // block exclusive scan of the counts
        OffT incl = cnt;
#pragma unroll
        for (int d = 1; d < kWarp; d <<= 1) {
            const OffT o = shfl_up(incl, d);
            if (lane >= d) incl += o;
        }
        if (lane == kWarp - 1) s_wsum[warp] = incl;
#pragma unroll
        for (int w = 0; w < NW; ++w) s_acc[w][tid] = 0.0;
        __syncthreads();
        OffT wpre = 0;
        for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
        OffT total = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) total += s_wsum[w];
        s_excl[tid] = wpre + incl - cnt;
        const int64_t base = (int64_t)A.off[tb];
        __syncthreads();
        // (the pipelined long-block loop of k_group_warp costs this kernel an
        // occupancy step on short rows, 0.22 -> 0.25 ms on C2u, so it stays plain)
        auto steps = [&](auto uc) {
          constexpr int U = decltype(uc)::value;
          SingleTileRun run;
          for (OffT k0 = 0; k0 < total; k0 += U * NT) {
            double p[U];
            gather_steps<ValT, U, NT>(A, x, base, k0, tid, total, p);
            if (LW_G_SINGLE == 1 && U > 1) {   // single-tile iteration (inside a long row)
                int t0 = 0;
#pragma unroll
                for (int s = NT / 2; s >= 1; s >>= 1)
                    if (t0 + s < tc && s_excl[t0 + s] <= k0) t0 += s;
                const OffT end = t0 + 1 < tc ? s_excl[t0 + 1] : total;
                const OffT last = k0 + (OffT)(U * NT) < total ? k0 + (OffT)(U * NT) : total;
                if (end >= last) {
                    run.take<U>(t0, p, lane, s_acc[warp]);
                    if (PROBE) {
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (k0 + u * NT + tid < total) { probe_atom(probe, base + k0 + u * NT + tid, glane, tb + t0); ++mine; }
                    }
                    continue;
                }
                run.flush(lane, s_acc[warp]);
            }
            int ts[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const OffT k = k0 + u * NT + tid;
                int t = 0;
                if (k < total) {
#pragma unroll
                    for (int s = NT / 2; s >= 1; s >>= 1)
                        if (t + s < tc && s_excl[t + s] <= k) t += s;
                }
                ts[u] = t;
                if (PROBE && k < total) { probe_atom(probe, base + k, glane, tb + t); ++mine; }
            }
            if (LW_G_SINGLE == 2 && U > 1) {
                // this warp's atoms of the iteration all in one tile (inside a long
                // row): no segmented reductions, a per-lane running sum instead
                const int tt = shfl(ts[0], 0);
                bool same = true;
#pragma unroll
                for (int u = 0; u < U; ++u) same = same && (k0 + u * NT + tid >= total || ts[u] == tt);
                if (__all_sync(0xffffffffu, same)) {
                    run.take<U>(tt, p, lane, s_acc[warp]);
                    continue;
                }
                run.flush(lane, s_acc[warp]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const OffT k = k0 + u * NT + tid;
                const bool valid = k < total;
                const int t = ts[u];
                const int key = valid ? t : INT_MAX;
                const int prev = shfl_up(key, 1);
                const bool head = lane == 0 || prev != key;
                const uint32_t heads = __ballot_sync(0xffffffffu, head);
                // a step's partial sums (<= 32 products) in the value precision
                const double sum = (double)warp_segsum_heads<ValT>((ValT)p[u], lane, heads);
                if (valid && head) s_acc[warp][t] += sum;
                __syncwarp();
            }
          }
          run.flush(lane, s_acc[warp]);
        };
        if (total >= (OffT)(GU_LONG * NT)) steps(std::integral_constant<int, GU>{});
        else steps(std::integral_constant<int, 1>{});
        __syncthreads();
        if (tid < tc) {
            double r = 0.0;
#pragma unroll
            for (int w = 0; w < NW; ++w) r += s_acc[w][tid];
            y[tb + tid] = (ValT)r;
        }
        __syncthreads();
    }
    if (PROBE && probe.lane_atoms) probe.lane_atoms[glane] = mine;
}

// ---- general groups -----------------------------------------------------------------
template <class ValT>
__device__ __forceinline__ void add_out(ValT* p, double v);
template <>
__device__ __forceinline__ void add_out<float>(float* p, double v) { atomicAdd(p, (float)v); }
template <>
__device__ __forceinline__ void add_out<double>(double* p, double v) { atomicAdd(p, v); }

template <class OffT, class ValT, bool PROBE>
__global__ void __launch_bounds__(256)
    k_group_generic(Csr<OffT, ValT> A, const ValT* __restrict__ x, ValT* __restrict__ y,
                    int64_t lanes, int64_t gs, int64_t tpb, Probe probe) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= lanes) return;
    const int64_t gid = l / gs, m = l - gid * gs;
    const int64_t members = min(gs, lanes - gid * gs);
    const int64_t groups = (lanes + gs - 1) / gs;
    const int64_t nblocks = (A.rows + tpb - 1) / tpb;
    int64_t mine = 0;
    for (int64_t b = gid; b < nblocks; b += groups) {
        const int64_t tb = b * tpb;
        const int64_t tc = min(tpb, A.rows - tb);
        const int64_t base = ld_off(A.off + tb);
        const int64_t total = ld_off(A.off + tb + tc) - base;
        int64_t tile = tb, cur = -1;
        double acc = 0.0;
        for (int64_t k = m; k < total; k += members) {
            const int64_t a = base + k;
            while (ld_off(A.off + tile + 1) <= a) ++tile;
            if (tile != cur) {
                if (cur >= 0) add_out<ValT>(y + cur, acc);
                cur = tile;
                acc = 0.0;
            }
            acc = fma((double)__ldg(A.val + a), (double)ld_gather(x + __ldg(A.col + a)), acc);
            if (PROBE) { probe_atom(probe, a, l, tile); ++mine; }
        }
        if (cur >= 0) add_out<ValT>(y + cur, acc);
    }
    if (PROBE && probe.lane_atoms) probe.lane_atoms[l] = mine;
}

// ---- general groups: y in the reference's member-major order ---------------------------
// The reference accumulates y[tile] += v*x member by member (_fast.py:66-77): member
// 0's atoms of the tile in increasing order, then member 1's, ... in fp64. One
// thread per tile replays exactly that order (MemberMajorWalk, lw_common.cuh) with
// unfused fp64 multiply and add, GT_U positions' loads in flight at a time. y is therefore run-to-run identical and, for fp64 data,
// bit-identical to the reference's spmv (tests: golden group configs compared
// exactly); no atomics, no zeroing pass. The lane -> atom mapping of these shapes
// is what k_group_generic executes (probe runs, which then rewrite y with this).
constexpr int GT_U = 8;   // positions per residue batch (loads in flight)
template <class OffT, class ValT>
__global__ void __launch_bounds__(256)
    k_group_tiles(Csr<OffT, ValT> A, const ValT* __restrict__ x, ValT* __restrict__ y, int64_t lanes,
                  int64_t gs, int64_t tpb) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= A.rows) return;
    const int64_t groups = (lanes + gs - 1) / gs;
    const int64_t b = t / tpb, g = b % groups;
    const int64_t M = min(gs, lanes - g * gs);   // members of the group owning block b
    const int64_t base = ld_off(A.off + b * tpb);
    const int64_t e0 = ld_off(A.off + t) - base, e1 = ld_off(A.off + t + 1) - base;
    double acc = 0.0;
    if (e1 - e0 >= GT_U * M) {
        // long tile: member by member (same order), GT_U of a member's positions
        // (stride M) in flight per batch, no walker arithmetic per position
        const int64_t r0 = e0 % M;
        auto member = [&](int64_t i) {
            for (int64_t k0 = e0 + i; k0 < e1; k0 += GT_U * M) {
                int32_t c[GT_U];
                double v[GT_U], xv[GT_U];
#pragma unroll
                for (int u = 0; u < GT_U; ++u) {
                    const int64_t k = k0 + u * M < e1 ? k0 + u * M : k0;
                    c[u] = __ldg(A.col + base + k);
                    v[u] = (double)__ldg(A.val + base + k);
                }
#pragma unroll
                for (int u = 0; u < GT_U; ++u) xv[u] = (double)ld_gather(x + c[u]);
#pragma unroll
                for (int u = 0; u < GT_U; ++u)
                    if (k0 + u * M < e1) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
            }
        };
        for (int64_t i = M - r0; i < M; ++i) member(i);   // wrapped residues 0, 1, ... first
        for (int64_t i = 0; i < M - r0; ++i) member(i);
        y[t] = (ValT)acc;
        return;
    }
    MemberMajorWalk w(e0, e1, M);
    for (int64_t p0 = w.next(); p0 >= 0;) {   // GT_U positions' loads in flight, then the ordered adds
        int64_t k[GT_U];
        k[0] = p0;
#pragma unroll
        for (int u = 1; u < GT_U; ++u) k[u] = k[u - 1] >= 0 ? w.next() : -1;
        int32_t c[GT_U];
        double v[GT_U], xv[GT_U];
#pragma unroll
        for (int u = 0; u < GT_U; ++u) {
            c[u] = k[u] >= 0 ? __ldg(A.col + base + k[u]) : 0;
            v[u] = k[u] >= 0 ? (double)__ldg(A.val + base + k[u]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < GT_U; ++u) xv[u] = k[u] >= 0 ? (double)ld_gather(x + c[u]) : 0.0;
#pragma unroll
        for (int u = 0; u < GT_U; ++u)
            if (k[u] >= 0) acc = __dadd_rn(acc, __dmul_rn(v[u], xv[u]));
        p0 = k[GT_U - 1] >= 0 ? w.next() : -1;
    }
    y[t] = (ValT)acc;
}

// ---- host side ----------------------------------------------------------------------
enum GroupKernel { GK_WARP, GK_BLOCK, GK_GENERIC };

static GroupKernel pick_group_kernel(int64_t lanes, int64_t gs, int64_t tpb) {
    if (gs == 32 && tpb == 32 && lanes % 32 == 0) return GK_WARP;
    if (gs == tpb && (gs == 64 || gs == 128 || gs == 256) && lanes % gs == 0) return GK_BLOCK;
    return GK_GENERIC;
}

// Groups one SM holds at once for the warp / block kernels (their register use,
// not 2048 threads, sets it), so the auto lane count is one full wave.
template <class K>
static int64_t resident_ctas(K kern, int nt) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, nt, 0) != cudaSuccess || n < 1) return 0;
    return n;
}
static int64_t groups_per_sm(int64_t gs, int64_t tpb) {
#ifndef LW_GROUP_OCC
#define LW_GROUP_OCC 1
#endif
    if (LW_GROUP_OCC) {
        if (gs == 32 && tpb == 32) {
            // both launches of the staged/cooperative pair run the same groups: size
            // them to the kernel with fewer resident CTAs, one wave for each
            static const int64_t w = std::min(
                resident_ctas(k_group_warp<int32_t, float, false, (LW_GW_CAP > 0 ? GW_STAGED : GW_ALL)>, 256),
                resident_ctas(k_group_warp<int32_t, float, false, (LW_GW_CAP > 0 ? GW_COOP : GW_ALL)>, 256)) * 8;
            if (w > 0) return w;
        } else if (gs == tpb && (gs == 256 || gs == 128 || gs == 64)) {
            // one resident wave of the launched (fused) kernel
#define LW_GB_OCC(NT) resident_ctas(k_group_block<int32_t, float, NT, false, (LW_GB_CAP > 0 ? GB_FUSED : GB_ALL)>, NT)
            static const int64_t b256 = LW_GB_OCC(256), b128 = LW_GB_OCC(128), b64 = LW_GB_OCC(64);
#undef LW_GB_OCC
            const int64_t b = gs == 256 ? b256 : gs == 128 ? b128 : b64;
            if (b > 0) return b;
        }
    }
    return gs < 2048 ? 2048 / gs : 1;
}

int64_t group_auto_lanes(int64_t rows, int64_t gs, int64_t tpb) {
    const int64_t nblocks = rows > 0 ? ceil_div(rows, tpb) : 1;
    // enough groups to fill every SM once, but never more than blocks
    const int64_t per_sm = groups_per_sm(gs, tpb);
    const int64_t cap = (int64_t)sm_count() * per_sm;
    const int64_t groups = nblocks < cap ? nblocks : cap;
    return (groups > 0 ? groups : 1) * gs;
}

template <class OffT, class ValT>
static int launch_group(const lw_csr_t* A, const void* x, void* y, int64_t lanes, int64_t gs,
                        int64_t tpb, const lw_probe_t* probe, cudaStream_t s) {
    Csr<OffT, ValT> a{A->rows, A->cols, A->nnz, (const OffT*)A->row_offsets,
                      A->col_indices, (const ValT*)A->values};
    Probe p{};
    if (probe) p = Probe{probe->lane_atoms, probe->atom_lane, probe->atom_tile, probe->atom_visits};
    if (probe && p.lane_atoms) LW_TRY(cudaMemsetAsync(p.lane_atoms, 0, lanes * 8, s));
    const ValT* xv = (const ValT*)x;
    ValT* yv = (ValT*)y;
    switch (pick_group_kernel(lanes, gs, tpb)) {
        case GK_WARP: {
            const int64_t groups = lanes / 32;
            const int64_t grid = ceil_div(groups, 8);
            if (probe) {
                k_group_warp<OffT, ValT, true><<<grid, 256, 0, s>>>(a, xv, yv, groups, p);
            } else if (LW_GW_CAP > 0 && ceil_div(A->rows, 32) >= 4 * (int64_t)sm_count()) {
                // (a few hundred blocks: one launch of the cooperative kernel is faster,
                // C1 0.053 vs 0.087 ms for the staged/cooperative pair)
                k_group_warp<OffT, ValT, false, GW_STAGED><<<grid, 256, 0, s>>>(a, xv, yv, groups, p);
                LW_LAUNCH_CHECK();
                k_group_warp<OffT, ValT, false, GW_COOP><<<grid, 256, 0, s>>>(a, xv, yv, groups, p);
            } else {
                k_group_warp<OffT, ValT, false><<<grid, 256, 0, s>>>(a, xv, yv, groups, p);
            }
            break;
        }
        case GK_BLOCK: {
            const int64_t groups = lanes / gs;
#define LW_GB(NT)                                                                           \
    if (gs == NT) {                                                                         \
        if (probe) {                                                                        \
            k_group_block<OffT, ValT, NT, true><<<groups, NT, 0, s>>>(a, xv, yv, groups, p); \
        } else if (LW_GB_CAP > 0) {                                                         \
            k_group_block<OffT, ValT, NT, false, GB_FUSED><<<groups, NT, 0, s>>>(a, xv, yv, groups, p); \
        } else {                                                                            \
            k_group_block<OffT, ValT, NT, false><<<groups, NT, 0, s>>>(a, xv, yv, groups, p); \
        }                                                                                   \
    }
            LW_GB(64) LW_GB(128) LW_GB(256)
#undef LW_GB
            break;
        }
        default: {
            if (probe) {   // the lane -> atom instrumentation, then y in the reference order
                LW_TRY(cudaMemsetAsync(y, 0, A->rows * sizeof(ValT), s));
                k_group_generic<OffT, ValT, true><<<ceil_div(lanes, 256), 256, 0, s>>>(a, xv, yv, lanes, gs, tpb, p);
                LW_LAUNCH_CHECK();
            }
            k_group_tiles<OffT, ValT><<<ceil_div(A->rows, 256), 256, 0, s>>>(a, xv, yv, lanes, gs, tpb);
        }
    }
    LW_LAUNCH_CHECK();
    return LW_OK;
}

int spmv_group_mapped(const lw_csr_t* A, const void* x, void* y, int64_t lanes, int64_t gs,
                      int64_t tpb, const lw_probe_t* probe, cudaStream_t s) {
    if (A->rows == 0) return LW_OK;
    const bool o32 = A->offset_bits == 32;
    if (A->dtype == LW_F32)
        return o32 ? launch_group<int32_t, float>(A, x, y, lanes, gs, tpb, probe, s)
                   : launch_group<int64_t, float>(A, x, y, lanes, gs, tpb, probe, s);
    return o32 ? launch_group<int32_t, double>(A, x, y, lanes, gs, tpb, probe, s)
               : launch_group<int64_t, double>(A, x, y, lanes, gs, tpb, probe, s);
}

// Group plan prefix of every block: prefix[b*(tpb+1)+i] = off[tb+min(i,tc)] - off[tb].
template <class OffT>
__global__ void k_group_prefix(const OffT* __restrict__ off, int64_t rows, int64_t tpb,
                               int64_t nblocks, int64_t* __restrict__ prefix) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nblocks * (tpb + 1)) return;
    const int64_t b = idx / (tpb + 1), i = idx - b * (tpb + 1);
    const int64_t tb = b * tpb;
    const int64_t tc = min(tpb, rows - tb);
    prefix[idx] = ld_off(off + tb + min(i, tc)) - ld_off(off + tb);
}

int group_plan_prefix(int64_t rows, const void* off, int bits, int64_t tpb, int64_t* prefix,
                      cudaStream_t s) {
    if (tpb < 1 || rows < 0 || !prefix) return LW_E_INVALID_ARG;
    if (rows == 0) return LW_OK;
    const int64_t nblocks = ceil_div(rows, tpb);
    const int64_t n = nblocks * (tpb + 1);
    if (bits == 32) k_group_prefix<int32_t><<<ceil_div(n, 256), 256, 0, s>>>((const int32_t*)off, rows, tpb, nblocks, prefix);
    else            k_group_prefix<int64_t><<<ceil_div(n, 256), 256, 0, s>>>((const int64_t*)off, rows, tpb, nblocks, prefix);
    LW_LAUNCH_CHECK();
    return LW_OK;
}

}  // namespace lw
