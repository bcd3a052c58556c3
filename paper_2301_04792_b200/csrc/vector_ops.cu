// vector_ops.cu — the power iteration's normalisation (BASELINE C5): ||y||_2 with a
// deterministic two-level fp64 reduction, and x = y / ||y|| in one pass.
//
// The reference-side driver (distributed.power_iteration) used torch for these,
// which costs about four passes over y per iteration (0.85 ms at 2^26 rows,
// 15% of the iteration). Here: one read of y for the norm (fixed per-CTA
// segments reduced in a fixed order, so the result is run-to-run identical) and
// one read + one write for the scaling.
#include <algorithm>

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
    for (int64_t i = b0 + threadIdx.x; i < b1; i += VO_NT) {
        const double v = (double)__ldg(y + i);
        acc = fma(v, v, acc);
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
__global__ void k_scale(const ValT* __restrict__ y, int64_t n, const double* __restrict__ norm,
                        ValT* __restrict__ x) {
    const double nrm = norm[0];
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const ValT v = y[i];
        x[i] = nrm > 0.0 ? (ValT)((double)v / nrm) : v;
    }
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
    if (dtype == LW_F32) k_scale<float><<<grid, 256, 0, s>>>((const float*)y, n, norm, (float*)x);
    else k_scale<double><<<grid, 256, 0, s>>>((const double*)y, n, norm, (double*)x);
    LW_LAUNCH_CHECK();
    return LW_OK;
}

}  // namespace lw
