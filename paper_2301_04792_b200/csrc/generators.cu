// generators.cu — counter-based synthetic inputs built on the device.
//
// The reference only ships NumPy generators for uniform and Zipf-length
// matrices (sparse.py:164-223). The north star's C2b/C3/C5 configs need banded
// and R-MAT matrices at up to 2^26 rows, far beyond what a Python loop builds,
// so the keys and values are pure functions of (seed, counter) defined in
// include/lw_hash.h: this file and oracle/lw_oracle.c evaluate the same
// functions and therefore produce identical CSR matrices.
#include "lw_common.cuh"
#include "lw_hash.h"

namespace lw {

__global__ void k_rmat_keys(int scale, int64_t edge_begin, int64_t n_edges, uint32_t t_a,
                            uint32_t t_ab, uint32_t t_abc, uint64_t seed,
                            int64_t* __restrict__ keys) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_edges; i += stride)
        keys[i] = (int64_t)lw_rmat_key(seed, (uint64_t)(edge_begin + i), scale, t_a, t_ab, t_abc);
}

__global__ void k_uniform_keys(uint64_t space, int64_t begin, int64_t n, uint64_t seed,
                               int64_t* __restrict__ keys) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        keys[i] = (int64_t)lw_uniform_key(seed, (uint64_t)(begin + i), space);
}

template <class ValT>
__global__ void k_hash_values(const int64_t* __restrict__ keys, int64_t n, uint64_t seed,
                              ValT* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] = (ValT)lw_hash_value(seed, (uint64_t)keys[i]);
}

int rmat_keys(int scale, int64_t edge_begin, int64_t n_edges, uint32_t t_a, uint32_t t_ab, uint32_t t_abc,
              uint64_t seed, int64_t* keys, cudaStream_t s) {
    if (scale < 1 || scale > 31 || n_edges < 0 || edge_begin < 0 || (!keys && n_edges > 0) || !(t_a <= t_ab && t_ab <= t_abc))
        return LW_E_INVALID_ARG;
    if (n_edges == 0) return LW_OK;
    const int64_t grid = min(ceil_div(n_edges, 256), (int64_t)sm_count() * 16);
    k_rmat_keys<<<grid, 256, 0, s>>>(scale, edge_begin, n_edges, t_a, t_ab, t_abc, seed, keys);
    LW_LAUNCH_CHECK();
    return LW_OK;
}

int uniform_keys(int64_t space, int64_t begin, int64_t n, uint64_t seed, int64_t* keys, cudaStream_t s) {
    if (space < 1 || n < 0 || begin < 0 || (!keys && n > 0)) return LW_E_INVALID_ARG;
    if (n == 0) return LW_OK;
    const int64_t grid = min(ceil_div(n, 256), (int64_t)sm_count() * 16);
    k_uniform_keys<<<grid, 256, 0, s>>>((uint64_t)space, begin, n, seed, keys);
    LW_LAUNCH_CHECK();
    return LW_OK;
}

int hash_values(const int64_t* keys, int64_t n, uint64_t seed, int dtype, void* out,
                cudaStream_t s) {
    if (n < 0 || (n > 0 && (!keys || !out))) return LW_E_INVALID_ARG;
    if (n == 0) return LW_OK;
    const int64_t grid = min(ceil_div(n, 256), (int64_t)sm_count() * 16);
    if (dtype == LW_F32) k_hash_values<float><<<grid, 256, 0, s>>>(keys, n, seed, (float*)out);
    else if (dtype == LW_F64) k_hash_values<double><<<grid, 256, 0, s>>>(keys, n, seed, (double*)out);
    else return LW_E_INVALID_ARG;
    LW_LAUNCH_CHECK();
    return LW_OK;
}

}  // namespace lw
