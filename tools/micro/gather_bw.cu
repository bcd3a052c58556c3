// Microbenchmark: the B200's ceiling for the SpMV access pattern without the
// reduction logic. Each thread streams IPT consecutive (col, val) with 32-byte
// loads, gathers x[col] (L2-resident x), and writes one partial sum per thread.
#include <cstdint>
#include <cuda_runtime.h>

template <int IPT, bool GATHER>
__global__ void __launch_bounds__(256) k_gather(const int* __restrict__ col, const float* __restrict__ val,
                                                const float* __restrict__ x, float* __restrict__ out,
                                                long n) {
    long i0 = ((long)blockIdx.x * blockDim.x + threadIdx.x) * IPT;
    if (i0 + IPT > n) return;
    int c[IPT];
    float v[IPT];
#pragma unroll
    for (int h = 0; h < IPT; h += 8) {
        asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(c[h]), "=r"(c[h + 1]), "=r"(c[h + 2]), "=r"(c[h + 3]), "=r"(c[h + 4]),
                       "=r"(c[h + 5]), "=r"(c[h + 6]), "=r"(c[h + 7])
                     : "l"(col + i0 + h));
        asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(v[h]), "=f"(v[h + 1]), "=f"(v[h + 2]), "=f"(v[h + 3]), "=f"(v[h + 4]),
                       "=f"(v[h + 5]), "=f"(v[h + 6]), "=f"(v[h + 7])
                     : "l"(val + i0 + h));
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < IPT; ++k) s += v[k] * (GATHER ? __ldg(x + c[k]) : (float)c[k]);
    out[i0 / IPT] = s;
}

extern "C" int gather_bw(int mode, const int* col, const float* val, const float* x, float* out, long n,
                         cudaStream_t s) {
    const int NT = 256;
    if (mode == 0) k_gather<16, true><<<(n / 16 + NT - 1) / NT, NT, 0, s>>>(col, val, x, out, n);
    else if (mode == 1) k_gather<16, false><<<(n / 16 + NT - 1) / NT, NT, 0, s>>>(col, val, x, out, n);
    else if (mode == 2) k_gather<8, true><<<(n / 8 + NT - 1) / NT, NT, 0, s>>>(col, val, x, out, n);
    else k_gather<32, true><<<(n / 32 + NT - 1) / NT, NT, 0, s>>>(col, val, x, out, n);
    return (int)cudaGetLastError();
}
