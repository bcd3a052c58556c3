// Microbenchmark: can TMA gather4 (sm_100 `cp.async.bulk.tensor.2d ... tile::gather4`)
// serve x gathers beside the LSU path and lift the C3 request ceiling?
// Same access pattern as gather_bw.cu: one-shot CTAs, each thread streams IPT=8
// consecutive (col, val) with 32-byte loads, gathers x, writes one partial sum.
// NTMA of a thread's 8 gathers go through TMA: x is viewed as a 2D tensor of
// 16-byte rows ([cols/4][4] fp32), one gather4 fetches the 4 rows col>>2 of 4
// atoms into 64 B of shared memory, completion on one mbarrier per CTA; the
// other 8-NTMA gathers are ordinary ld.global.nc loads.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>

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

template <int NT, int NTMA>
__global__ void __launch_bounds__(NT) k_tg(const __grid_constant__ CUtensorMap tm, const int* __restrict__ col,
                                           const float* __restrict__ val, const float* __restrict__ x,
                                           float* __restrict__ out, long nseg) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t mbar;
    const long seg = blockIdx.x;
    if (seg >= nseg) return;
    const int tid = threadIdx.x;
    const long i0 = (seg * NT + tid) * 8;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&mbar);
    if (NTMA > 0 && tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(NT));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    int c[8];
    float v[8], g[8];
    ld8c(col + i0, c);
    ld8v(val + i0, v);
    if (NTMA > 0) __syncthreads();
    const uint32_t slot = (uint32_t)__cvta_generic_to_shared(sm) + (uint32_t)tid * (NTMA / 4) * 128u;
    if (NTMA > 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(NTMA * 16)
                     : "memory");
#pragma unroll
        for (int q = 0; q < NTMA / 4; ++q) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(slot + 128u * q),
                "l"(&tm), "r"(0), "r"(c[4 * q] >> 2), "r"(c[4 * q + 1] >> 2), "r"(c[4 * q + 2] >> 2),
                "r"(c[4 * q + 3] >> 2), "r"(bar)
                : "memory");
        }
    }
#pragma unroll
    for (int k = NTMA; k < 8; ++k) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(g[k]) : "l"(x + c[k]));
    if (NTMA > 0) {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done) : "r"(bar) : "memory");
        }
#pragma unroll
        for (int k = 0; k < NTMA; ++k) {
            const uint32_t a = slot + 128u * (k / 4) + 16u * (k % 4) + 4u * (uint32_t)(c[k] & 3);
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(g[k]) : "r"(a));
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k] * g[k];
    out[seg * NT + tid] = acc;
}

// ntma = -1: "transposed" atom order — gather instruction k of a warp reads the
// 32 consecutive atoms 32k + lane of the warp's 256-atom block (sorted columns of
// one row sit side by side in one instruction), instead of atom 8*lane + k.
template <int NT>
__global__ void __launch_bounds__(NT) k_tr(const int* __restrict__ col, const float* __restrict__ val,
                                           const float* __restrict__ x, float* __restrict__ out, long nseg) {
    const long seg = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long b = (seg * NT + warp * 32) * 8;
    int c[8];
    float v[8], g[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(c[k]) : "l"(col + b + 32 * k + lane));
        asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v[k]) : "l"(val + b + 32 * k + lane));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(g[k]) : "l"(x + c[k]));
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += v[k] * g[k];
    out[seg * NT + threadIdx.x] = acc;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

template <int NT, int NTMA>
static int launch(const CUtensorMap& tm, const int* col, const float* val, const float* x, float* out, long nseg,
                  cudaStream_t s) {
    auto kern = k_tg<NT, NTMA>;
    const int smem = NT * (NTMA / 4) * 128;
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<(unsigned)nseg, NT, smem, s>>>(tm, col, val, x, out, nseg);
    return (int)cudaGetLastError();
}

// n atoms (multiple of 8*nt); x has cols fp32 (multiple of 4). Returns a cudaError / CUresult code.
extern "C" int tma_gather(int nt, int ntma, const int* col, const float* val, const float* x, long cols,
                          float* out, long n, cudaStream_t s) {
    CUtensorMap tm;
    auto fn = encode();
    if (!fn) return -1;
    cuuint64_t dims[2] = {4, (cuuint64_t)(cols / 4)};
    cuuint64_t strides[1] = {16};
    cuuint32_t box[2] = {4, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)x, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return 1000 + (int)r;
    const long nseg = n / (8L * nt);
    if (ntma == -1 && nt == 512) {
        k_tr<512><<<(unsigned)nseg, 512, 0, s>>>(col, val, x, out, nseg);
        return (int)cudaGetLastError();
    }
#define LW_TG(NT_, K_) \
    if (nt == NT_ && ntma == K_) return launch<NT_, K_>(tm, col, val, x, out, nseg, s);
    LW_TG(512, 0) LW_TG(512, 4) LW_TG(512, 8) LW_TG(256, 0) LW_TG(256, 4) LW_TG(256, 8) LW_TG(128, 4)
    LW_TG(128, 8)
#undef LW_TG
    return -2;
}
