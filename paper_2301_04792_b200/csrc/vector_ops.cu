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

// x = y / ||y|| per element, rounded like (ValT)((double)y / nrm).
// fp32: the fp64 quotient by Markstein's correction of a reciprocal multiply —
// inv = RN(1/b) (one IEEE division per thread), q0 = RN(a*inv), r = a - b*q0
// (exact by FMA), q = RN(q0 + r*inv) — which is RN(a/b) whenever inv is the
// correctly rounded reciprocal and no intermediate leaves the normal range
// (Markstein 1990; the IEEE fp64 divide does the same plus a slow path for
// range extremes). Here a is an fp32 value widened to fp64 (|a| < 2^128) and b a
// norm of fp32 values (2^-149 <= b < 2^141), so q0, r and r*inv stay far inside
// fp64's normal range: the result is bit-identical to the division
// (tests/test_gpu_parity.py checks it over every fp32 exponent). Non-finite a
// gives a NaN residual and a = +-0 a +0 correction; q0 (= a / b for inf, NaN
// and signed zeros) is returned then.
// fp64 keeps the IEEE division (a may be tiny enough for r to underflow).
template <class ValT>
__device__ __forceinline__ ValT div_norm(ValT v, double b, double inv) {
    if constexpr (sizeof(ValT) == 4) {
        const double a = (double)v;
        const double q0 = a * inv;
        const double q = fma(fma(-q0, b, a), inv, q0);
        return (ValT)(q == q && q0 != 0.0 ? q : q0);
    } else {
        return (ValT)((double)v / b);
    }
}

// 16-byte vectors (4 fp32 / 2 fp64), U of them per thread in flight before the
// first divide (one vector per thread left the loop latency-bound: 215 us for
// 2^26 fp32 in the C5 loop, 2.4 TB/s).
template <class ValT>
__global__ void __launch_bounds__(256) k_scale_vec(const ValT* y, int64_t n, const double* __restrict__ norm,
                                                   ValT* x) {   // x may be y
    constexpr int V = 16 / sizeof(ValT), U = 4;
    using Vec = typename std::conditional<sizeof(ValT) == 4, float4, double2>::type;
    const double b = norm[0];
    if (!(b > 0.0)) {   // y = 0: x = y
        if (x == y) return;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
            x[i] = y[i];
        return;
    }
    const double inv = 1.0 / b;
    const int64_t nv = n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < nv; i += U * stride) {
        Vec v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = reinterpret_cast<const Vec*>(y)[i + u * stride];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            ValT* e = reinterpret_cast<ValT*>(&v[u]);
#pragma unroll
            for (int k = 0; k < V; ++k) e[k] = div_norm(e[k], b, inv);
            reinterpret_cast<Vec*>(x)[i + u * stride] = v[u];
        }
    }
    for (; i < nv; i += stride) {
        Vec v = reinterpret_cast<const Vec*>(y)[i];
        ValT* e = reinterpret_cast<ValT*>(&v);
#pragma unroll
        for (int k = 0; k < V; ++k) e[k] = div_norm(e[k], b, inv);
        reinterpret_cast<Vec*>(x)[i] = v;
    }
    const int64_t t = nv * V + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // tail
    if (t < n) x[t] = div_norm(y[t], b, inv);
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
                                                                          (int64_t)sm_count() * 8));
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
