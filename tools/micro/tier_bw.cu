// Microbenchmark: does a shared-memory (or cluster DSMEM) tier for the hottest
// x values lift the C3 gather ceiling?  Same access pattern as gather_bw.cu
// (stream IPT consecutive (col, val) with 32-byte loads, gather x, one partial
// sum per thread), but hot columns are relabeled to slot | 0x80000000 and read
// from a copy of xh[0..K) held in shared memory:
//   mode 0: persistent CTAs, no tier (occupancy reference)
//   mode 1: persistent CTAs, each holding xh[0..K) in its own shared memory
//   mode 2: clusters of C CTAs; CTA r of a cluster holds slots s with s % C == r
//           at s / C, read across the cluster through DSMEM
// Segments of NT*IPT atoms are walked grid-stride, so concurrently running CTAs
// stay on neighbouring rows (the locality the non-persistent SpMV has).
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ void ld8c(const int* p, int* c) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(c[0]), "=r"(c[1]), "=r"(c[2]), "=r"(c[3]), "=r"(c[4]), "=r"(c[5]), "=r"(c[6]),
                   "=r"(c[7])
                 : "l"(p));
}
__device__ __forceinline__ void ld8v(const float* p, float* v) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
                   "=f"(v[7])
                 : "l"(p));
}
__device__ __forceinline__ float ld_cold(const float* p, int l1) {
    float v;
    if (l1) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
    else asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p));
    return v;
}

template <int IPT, int MODE, int C>
__global__ void k_tier(const int* __restrict__ col, const float* __restrict__ val, const float* __restrict__ x,
                       const float* __restrict__ xh, int k_local, float* __restrict__ out, long nseg, int l1) {
    extern __shared__ float s_x[];
    const int NT = blockDim.x;
    if (MODE == 1) {
        for (int i = threadIdx.x; i < k_local; i += NT) s_x[i] = xh[i];
        __syncthreads();
    }
    if (MODE == 2) {
        cg::cluster_group cl = cg::this_cluster();
        const int r = (int)cl.block_rank();
        for (int i = threadIdx.x; i < k_local; i += NT) s_x[i] = xh[(long)i * C + r];
        cl.sync();
    }
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(s_x);
    for (long seg = blockIdx.x; seg < nseg; seg += gridDim.x) {
        const long i0 = (seg * NT + threadIdx.x) * IPT;
        int c[IPT];
        float v[IPT], g[IPT];
#pragma unroll
        for (int h = 0; h < IPT; h += 8) { ld8c(col + i0 + h, c + h); ld8v(val + i0 + h, v + h); }
#pragma unroll
        for (int k = 0; k < IPT; ++k) {
            const int ck = c[k];
            if (MODE == 3) {   // dense hot prefix [0, k_local) kept in L1, the rest bypasses L1
                if (ck < k_local) asm volatile("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(g[k]) : "l"(x + ck));
                else asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(g[k]) : "l"(x + ck));
            } else if (MODE == 0 || ck >= 0) {
                g[k] = ld_cold(x + (ck & 0x7fffffff), l1);
            } else {
                const int s = ck & 0x7fffffff;
                if (MODE == 1) g[k] = s_x[s];
                else {
                    uint32_t ra;
                    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(s_base + 4u * (uint32_t)(s / C)), "r"(s & (C - 1)));
                    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(g[k]) : "r"(ra));
                }
            }
        }
        float acc = 0.f;
#pragma unroll
        for (int k = 0; k < IPT; ++k) acc += v[k] * g[k];
        out[seg * NT + threadIdx.x] = acc;
    }
    if (MODE == 2) cg::this_cluster().sync();   // keep my tier alive until the cluster is done
}

template <int IPT, int MODE, int C>
static int launch(int grid, int nt, size_t smem, const int* col, const float* val, const float* x,
                  const float* xh, int k_local, float* out, long nseg, int l1, cudaStream_t s) {
    auto kern = k_tier<IPT, MODE, C>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (MODE == 2) {
        if (C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(nt);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return (int)cudaLaunchKernelEx(&cfg, kern, col, val, x, xh, k_local, out, nseg, l1);
    }
    kern<<<grid, nt, smem, s>>>(col, val, x, xh, k_local, out, nseg, l1);
    return (int)cudaGetLastError();
}

// max active clusters of size C with this block / smem shape (0 on error)
template <int C>
static int max_clusters(int nt, size_t smem) {
    auto kern = k_tier<8, 2, C>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (C > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C * 16);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) return 0;
    return n;
}

extern "C" int tier_max_clusters(int C, int nt, long smem) {
    switch (C) {
        case 2: return max_clusters<2>(nt, smem);
        case 4: return max_clusters<4>(nt, smem);
        case 8: return max_clusters<8>(nt, smem);
        case 16: return max_clusters<16>(nt, smem);
    }
    return -1;
}

extern "C" int tier_bw(int mode, int C, int grid, int nt, long smem, const int* col, const float* val,
                       const float* x, const float* xh, int k_local, float* out, long n, int l1,
                       cudaStream_t s) {
    const long nseg = n / (8L * nt);
    if (mode == 0) return launch<8, 0, 1>(grid, nt, smem, col, val, x, xh, k_local, out, nseg, l1, s);
    if (mode == 3) return launch<8, 3, 1>(grid, nt, smem, col, val, x, xh, k_local, out, nseg, l1, s);
    if (mode == 1) return launch<8, 1, 1>(grid, nt, smem, col, val, x, xh, k_local, out, nseg, l1, s);
    switch (C) {
        case 2: return launch<8, 2, 2>(grid, nt, smem, col, val, x, xh, k_local, out, nseg, l1, s);
        case 4: return launch<8, 2, 4>(grid, nt, smem, col, val, x, xh, k_local, out, nseg, l1, s);
        case 8: return launch<8, 2, 8>(grid, nt, smem, col, val, x, xh, k_local, out, nseg, l1, s);
        case 16: return launch<8, 2, 16>(grid, nt, smem, col, val, x, xh, k_local, out, nseg, l1, s);
    }
    return -1;
}
