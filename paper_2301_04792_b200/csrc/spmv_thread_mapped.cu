// spmv_thread_mapped.cu — thread_mapped schedule: one tile (row) per lane.
//
// Schedule (reference schedules.py:57-60 -> work.py:85-92):
// lane l of P owns tiles l, l+P, l+2P, ... and each owned tile's full atom range.
// On the device a lane is one thread (lane = blockIdx.x*blockDim.x+threadIdx.x),
// so the per-lane tile sets are exactly the reference's and
// executor.imbalance(ts, cfg(P)) (executor.py:228-230) predicts per-thread work.
//
// Kernel (replaces _fast.spmv_thread_mapped, _fast.py:20-28): the row is walked
// with 128-bit loads of values and matching-width loads of col_idx after a scalar
// alignment prologue; products and sums are fp64; y[t] is assigned (not
// accumulated), so empty rows get 0 like the reference (kernels.py:63 + _fast.py:28).
#include "lw_common.cuh"

#ifndef LW_TM_UV
#define LW_TM_UV 4   // vectors in flight per thread on long rows
#endif
// rows of >= LW_TM_LONG * UV vectors take the pipelined loop: 48 atoms fp32, 16
// fp64 (8 / 8: C1 fp32 0.0246 -> 0.0164 ms, C2u fp64 0.235 -> 0.192, C2b fp32
// unchanged at 3 and +7% at 2)
#ifndef LW_TM_LONG
#define LW_TM_LONG 3
#endif
#ifndef LW_TM_WIDE   // A/B: the few-lanes instantiation with 2*UV vectors in flight
#define LW_TM_WIDE 1
#endif
#ifndef LW_TM_LONG64
#define LW_TM_LONG64 2
#endif

namespace lw {

template <class ValT>
struct VecTraits;
template <>
struct VecTraits<float> {
    static constexpr int V = 4;
    using ValV = float4;
    using ColV = int4;
};
template <>
struct VecTraits<double> {
    static constexpr int V = 2;
    using ValV = double2;
    using ColV = int2;
};

template <class ValT>
__device__ __forceinline__ void accum_vec(const typename VecTraits<ValT>::ValV& v,
                                          const typename VecTraits<ValT>::ColV& c,
                                          const ValT* __restrict__ x, double& a0,
                                          double& a1);
template <>
__device__ __forceinline__ void accum_vec<float>(const float4& v, const int4& c,
                                                 const float* __restrict__ x, double& a0,
                                                 double& a1) {
    float x0 = ld_gather(x + c.x), x1 = ld_gather(x + c.y);
    float x2 = ld_gather(x + c.z), x3 = ld_gather(x + c.w);
    a0 = fma((double)v.x, (double)x0, a0);
    a1 = fma((double)v.y, (double)x1, a1);
    a0 = fma((double)v.z, (double)x2, a0);
    a1 = fma((double)v.w, (double)x3, a1);
}
template <>
__device__ __forceinline__ void accum_vec<double>(const double2& v, const int2& c,
                                                  const double* __restrict__ x, double& a0,
                                                  double& a1) {
    double x0 = ld_gather(x + c.x), x1 = ld_gather(x + c.y);
    a0 = fma(v.x, x0, a0);
    a1 = fma(v.y, x1, a1);
}

// Dot product of row atoms [b, e) with x, fp64 accumulation in two chains.
template <class ValT, bool VEC, int UV, int LONG>
__device__ __forceinline__ double row_dot(const int32_t* __restrict__ col,
                                          const ValT* __restrict__ val,
                                          const ValT* __restrict__ x, int64_t b, int64_t e) {
    using VT = VecTraits<ValT>;
    constexpr int V = VT::V;
    double a0 = 0.0, a1 = 0.0;
    if (VEC) {
        while (b < e && (b & (V - 1)) != 0) {
            a0 = fma((double)__ldg(val + b), (double)ld_gather(x + __ldg(col + b)), a0);
            ++b;
        }
        // long rows: UV vectors per step, every load issued before the first use,
        // so a single thread keeps UV*V gathers in flight (the thread-mapped
        // schedule puts whole long rows on one thread)
        if (e - b >= LONG * UV * V) {   // only long rows; short rows keep the plain loop below
            // software pipeline: the next group's col_idx / values stream in
            // while this group's gathers are in flight, so a step costs one
            // round trip (the gathers) instead of two
            typename VT::ValV v[UV];
            typename VT::ColV c[UV];
#pragma unroll
            for (int u = 0; u < UV; ++u) {
                v[u] = __ldg(reinterpret_cast<const typename VT::ValV*>(val + b) + u);
                c[u] = __ldg(reinterpret_cast<const typename VT::ColV*>(col + b) + u);
            }
            for (; b + 2 * UV * V <= e; b += UV * V) {
                typename VT::ValV vn[UV];
                typename VT::ColV cn[UV];
#pragma unroll
                for (int u = 0; u < UV; ++u) {
                    vn[u] = __ldg(reinterpret_cast<const typename VT::ValV*>(val + b + UV * V) + u);
                    cn[u] = __ldg(reinterpret_cast<const typename VT::ColV*>(col + b + UV * V) + u);
                }
#pragma unroll
                for (int u = 0; u < UV; ++u) accum_vec<ValT>(v[u], c[u], x, a0, a1);
#pragma unroll
                for (int u = 0; u < UV; ++u) { v[u] = vn[u]; c[u] = cn[u]; }
            }
#pragma unroll
            for (int u = 0; u < UV; ++u) accum_vec<ValT>(v[u], c[u], x, a0, a1);
            b += UV * V;
        }
#pragma unroll 2
        for (; b + V <= e; b += V) {
            typename VT::ValV v = __ldg(reinterpret_cast<const typename VT::ValV*>(val + b));
            typename VT::ColV c = __ldg(reinterpret_cast<const typename VT::ColV*>(col + b));
            accum_vec<ValT>(v, c, x, a0, a1);
        }
    }
    for (; b < e; ++b)
        a1 = fma((double)__ldg(val + b), (double)ld_gather(x + __ldg(col + b)), a1);
    return a0 + a1;
}

// UV / LONG: vectors in flight per thread on rows of >= LONG*UV vectors. The sums
// do not depend on them (atoms are accumulated in order into the same two chains).
template <class OffT, class ValT, bool VEC, bool PROBE, int UV = LW_TM_UV,
          int LONG = (sizeof(ValT) == 4 ? LW_TM_LONG : LW_TM_LONG64)>
__global__ void __launch_bounds__(256)
    k_spmv_thread_mapped(Csr<OffT, ValT> A, const ValT* __restrict__ x,
                         ValT* __restrict__ y, int64_t lanes, Probe probe) {
    const int64_t lane = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (lane >= lanes) return;
    int64_t mine = 0;
    for (int64_t t = lane; t < A.rows; t += lanes) {
        const int64_t b = ld_off(A.off + t), e = ld_off(A.off + t + 1);
        y[t] = (ValT)row_dot<ValT, VEC, UV, LONG>(A.col, A.val, x, b, e);
        if (PROBE) {
            mine += e - b;
            for (int64_t a = b; a < e; ++a) probe_atom(probe, a, lane, t);
        }
    }
    if (PROBE && probe.lane_atoms) probe.lane_atoms[lane] = mine;
}

template <class OffT, class ValT>
int launch_thread_mapped(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                         const lw_probe_t* probe, cudaStream_t s) {
    Csr<OffT, ValT> a{A->rows, A->cols, A->nnz, (const OffT*)A->row_offsets,
                      A->col_indices, (const ValT*)A->values};
    // CTA size: 256 threads, or fewer when that leaves SMs idle — each lane is one
    // thread whatever the CTA size (same rows, same sums), but the lanes' gathers
    // then issue from every SM's L1 instead of a few (C1: 10 K lanes are 40 CTAs
    // of 256 on 40 of 148 SMs; at 64 they spread over all of them)
#ifndef LW_TM_SPREAD
#define LW_TM_SPREAD 1
#endif
    int NT = 256;
    if (LW_TM_SPREAD)
        while (NT > 32 && ceil_div(lanes, (int64_t)NT) < 2 * (int64_t)sm_count()) NT >>= 1;
    const int64_t grid = ceil_div(lanes, NT);
    if (grid > 0x7fffffff) return LW_E_UNSUPPORTED;
    const bool vec = ((uintptr_t)A->values % 16 == 0) && ((uintptr_t)A->col_indices % 16 == 0);
    Probe p{};
    if (probe) p = Probe{probe->lane_atoms, probe->atom_lane, probe->atom_tile, probe->atom_visits};
    if (probe && p.lane_atoms) LW_TRY(cudaMemsetAsync(p.lane_atoms, 0, lanes * 8, s));
    if (probe) {
        if (vec) k_spmv_thread_mapped<OffT, ValT, true, true><<<grid, NT, 0, s>>>(a, (const ValT*)x, (ValT*)y, lanes, p);
        else     k_spmv_thread_mapped<OffT, ValT, false, true><<<grid, NT, 0, s>>>(a, (const ValT*)x, (ValT*)y, lanes, p);
    } else if (vec && LW_TM_WIDE && lanes <= (int64_t)sm_count() * 128) {
        // few lanes (C1: 10 K rows): occupancy is not the limit, the per-thread
        // chain of gather round trips is, so each thread keeps twice the vectors
        // in flight from 2 groups on (same sums)
        k_spmv_thread_mapped<OffT, ValT, true, false, 2 * LW_TM_UV, 2><<<grid, NT, 0, s>>>(a, (const ValT*)x, (ValT*)y, lanes, p);
    } else {
        if (vec) k_spmv_thread_mapped<OffT, ValT, true, false><<<grid, NT, 0, s>>>(a, (const ValT*)x, (ValT*)y, lanes, p);
        else     k_spmv_thread_mapped<OffT, ValT, false, false><<<grid, NT, 0, s>>>(a, (const ValT*)x, (ValT*)y, lanes, p);
    }
    LW_LAUNCH_CHECK();
    return LW_OK;
}

int spmv_thread_mapped(const lw_csr_t* A, const void* x, void* y, int64_t lanes,
                       const lw_probe_t* probe, cudaStream_t s) {
    if (A->rows == 0) return LW_OK;
    const bool o32 = A->offset_bits == 32;
    if (A->dtype == LW_F32)
        return o32 ? launch_thread_mapped<int32_t, float>(A, x, y, lanes, probe, s)
                   : launch_thread_mapped<int64_t, float>(A, x, y, lanes, probe, s);
    return o32 ? launch_thread_mapped<int32_t, double>(A, x, y, lanes, probe, s)
               : launch_thread_mapped<int64_t, double>(A, x, y, lanes, probe, s);
}

}  // namespace lw
