// vector_ops.cu — the power iteration's normalisation (BASELINE C5): ||y||_2 with a
// deterministic two-level fp64 reduction, and x = y / ||y|| in one pass.
//
// The reference-side driver (distributed.power_iteration) used torch for these,
// which costs about four passes over y per iteration (0.85 ms at 2^26 rows,
// 15% of the iteration). Here: one read of y for the norm (fixed per-CTA
// segments reduced in a fixed order, so the result is run-to-run identical) and
// one read + one write for the scaling.
#include <algorithm>

#include <type_traits>

#include "lw_common.cuh"

namespace lw {

constexpr int VO_NT = 512;
constexpr int VO_ITEMS = 8192;   // elements per CTA segment

__device__ __forceinline__ double block_sum(double v, double* s_w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    if (lane == 0) s_w[warp] = v;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < VO_NT / 32 ? s_w[lane] : 0.0;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) t += __shfl_down_sync(0xffffffffu, t, d);
    }
    return t;   // valid in thread 0
}

template <class ValT>
__global__ void __launch_bounds__(VO_NT) k_sumsq_partials(const ValT* __restrict__ y, int64_t n,
                                                          double* __restrict__ partials) {
    __shared__ double s_w[VO_NT / 32];
    const int64_t b0 = (int64_t)blockIdx.x * VO_ITEMS;
    const int64_t b1 = min(b0 + VO_ITEMS, n);
    double acc = 0.0;
    constexpr int V = 16 / sizeof(ValT);                   // elements per 16-byte vector
    constexpr int PER = VO_ITEMS / VO_NT;                   // elements per thread (16)
    using Vec = typename std::conditional<sizeof(ValT) == 4, float4, double2>::type;
    if (b1 - b0 == VO_ITEMS && (uintptr_t)(y + b0) % 16 == 0) {
        // full segment: all PER/V vector loads in flight before the first FMA,
        // then a fixed accumulation order (run-to-run identical)
        const Vec* yv = reinterpret_cast<const Vec*>(y + b0);
        Vec r[PER / V];
#pragma unroll
        for (int h = 0; h < PER / V; ++h) r[h] = __ldg(yv + threadIdx.x + h * VO_NT);
#pragma unroll
        for (int h = 0; h < PER / V; ++h) {
            const ValT* e = reinterpret_cast<const ValT*>(&r[h]);
#pragma unroll
            for (int k = 0; k < V; ++k) acc = fma((double)e[k], (double)e[k], acc);
        }
    } else {
        for (int64_t i = b0 + threadIdx.x; i < b1; i += VO_NT) {
            const double v = (double)__ldg(y + i);
            acc = fma(v, v, acc);
        }
    }
    const double t = block_sum(acc, s_w);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

__global__ void __launch_bounds__(VO_NT) k_sumsq_final(const double* __restrict__ partials,
                                                       int64_t nb, double* __restrict__ out) {
    __shared__ double s_w[VO_NT / 32];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < nb; i += VO_NT) acc += partials[i];
    const double t = block_sum(acc, s_w);
    if (threadIdx.x == 0) out[0] = sqrt(t);
}

template <class ValT>
__global__ void k_scale(const ValT* y, int64_t n, const double* __restrict__ norm,
                        ValT* x) {   // x may be y (in-place scaling)
    const double nrm = norm[0];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const ValT v = y[i];
        x[i] = nrm > 0.0 ? (ValT)((double)v / nrm) : v;
    }
}

// The same per-element formula on 16-byte vectors (4 fp32 / 2 fp64 per load):
// independent divisions per thread keep the loads in flight (the scalar loop
// serialises load -> fp64 divide -> store). Results are identical.
template <class ValT>
__global__ void k_scale_vec(const ValT* y, int64_t n, const double* __restrict__ norm,
                            ValT* x) {   // x may be y
    constexpr int V = 16 / sizeof(ValT);
    using Vec = typename std::conditional<sizeof(ValT) == 4, float4, double2>::type;
    const double nrm = norm[0];
    const int64_t nv = n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
        Vec v = reinterpret_cast<const Vec*>(y)[i];
        ValT* e = reinterpret_cast<ValT*>(&v);
#pragma unroll
        for (int k = 0; k < V; ++k) e[k] = nrm > 0.0 ? (ValT)((double)e[k] / nrm) : e[k];
        reinterpret_cast<Vec*>(x)[i] = v;
    }
    const int64_t t = nv * V + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // tail
    if (t < n) x[t] = nrm > 0.0 ? (ValT)((double)y[t] / nrm) : y[t];
}

size_t norm_workspace(int64_t n) { return (size_t)(n > 0 ? ceil_div(n, VO_ITEMS) : 1) * 8; }

int vector_norm(const void* y, int64_t n, int dtype, void* ws, double* out, cudaStream_t s) {
    const int64_t nb = n > 0 ? ceil_div(n, VO_ITEMS) : 0;
    double* partials = (double*)ws;
    if (nb > 0) {
        if (dtype == LW_F32) k_sumsq_partials<float><<<(unsigned)nb, VO_NT, 0, s>>>((const float*)y, n, partials);
        else k_sumsq_partials<double><<<(unsigned)nb, VO_NT, 0, s>>>((const double*)y, n, partials);
        LW_LAUNCH_CHECK();
    }
    k_sumsq_final<<<1, VO_NT, 0, s>>>(partials, nb, out);
    LW_LAUNCH_CHECK();
    return LW_OK;
}

int vector_scale(const void* y, int64_t n, int dtype, const double* norm, void* x, cudaStream_t s) {
    if (n == 0) return LW_OK;
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, 256), (int64_t)sm_count() * 16);
    const bool vec = (uintptr_t)y % 16 == 0 && (uintptr_t)x % 16 == 0;
    if (vec) {
        const int64_t nv = n / (dtype == LW_F32 ? 4 : 2);
        const unsigned gv = (unsigned)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nv, 256),
                                                                          (int64_t)sm_count() * 16));
        if (dtype == LW_F32) k_scale_vec<float><<<gv, 256, 0, s>>>((const float*)y, n, norm, (float*)x);
        else k_scale_vec<double><<<gv, 256, 0, s>>>((const double*)y, n, norm, (double*)x);
    } else if (dtype == LW_F32) {
        k_scale<float><<<grid, 256, 0, s>>>((const float*)y, n, norm, (float*)x);
    } else {
        k_scale<double><<<grid, 256, 0, s>>>((const double*)y, n, norm, (double*)x);
    }
    LW_LAUNCH_CHECK();
    return LW_OK;
}

}  // namespace lw
