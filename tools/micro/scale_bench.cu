// x = y / nrm (fp64 divide, rounded to fp32) vs Markstein-corrected reciprocal multiply:
// time both on 2^24 / 2^26 fp32 vectors and count results that differ bit-wise.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_div(const float4* y, int64_t n4, const double* nrm, float4* x) {
    const double b = *nrm;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 v = y[i];
        v.x = (float)((double)v.x / b); v.y = (float)((double)v.y / b);
        v.z = (float)((double)v.z / b); v.w = (float)((double)v.w / b);
        x[i] = v;
    }
}
__device__ __forceinline__ double qdiv(double a, double b, double inv) {
    const double q0 = a * inv;
    const double r = fma(-q0, b, a);
    return fma(r, inv, q0);
}
__global__ void k_mul(const float4* y, int64_t n4, const double* nrm, float4* x) {
    const double b = *nrm, inv = 1.0 / b;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 v = y[i];
        v.x = (float)qdiv(v.x, b, inv); v.y = (float)qdiv(v.y, b, inv);
        v.z = (float)qdiv(v.z, b, inv); v.w = (float)qdiv(v.w, b, inv);
        x[i] = v;
    }
}
__global__ void k_cmp(const uint32_t* a, const uint32_t* b, int64_t n, unsigned long long* bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (a[i] != b[i]) atomicAdd(bad, 1ull);
}
__global__ void k_fill(float* y, int64_t n, uint64_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed; z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29;
        const uint32_t bits = (uint32_t)z;
        float f = __uint_as_float((bits & 0x807fffffu) | ((uint32_t)(100 + (z >> 40) % 56) << 23));
        y[i] = f;
    }
}
int main() {
    for (int sc : {24, 26}) {
        const int64_t n = 1ll << sc;
        float *y, *x1, *x2; double* nrm; unsigned long long* bad;
        cudaMalloc(&y, n * 4); cudaMalloc(&x1, n * 4); cudaMalloc(&x2, n * 4); cudaMalloc(&nrm, 8); cudaMalloc(&bad, 8);
        k_fill<<<148 * 16, 256>>>(y, n, 7);
        unsigned long long tot = 0;
        for (double b : {1.0, 3.0, 1234.5678, 0.0071, 7.3e5, 1.0 / 3.0, 9.87654321e-3}) {
            cudaMemcpy(nrm, &b, 8, cudaMemcpyHostToDevice);
            cudaMemset(bad, 0, 8);
            k_div<<<148 * 16, 256>>>((float4*)y, n / 4, nrm, (float4*)x1);
            k_mul<<<148 * 16, 256>>>((float4*)y, n / 4, nrm, (float4*)x2);
            k_cmp<<<148 * 16, 256>>>((uint32_t*)x1, (uint32_t*)x2, n, bad);
            unsigned long long h; cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost); tot += h;
        }
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        float t1, t2;
        for (int w = 0; w < 3; ++w) k_div<<<148 * 16, 256>>>((float4*)y, n / 4, nrm, (float4*)x1);
        cudaEventRecord(e0); for (int r = 0; r < 20; ++r) k_div<<<148 * 16, 256>>>((float4*)y, n / 4, nrm, (float4*)x1);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t1, e0, e1);
        for (int w = 0; w < 3; ++w) k_mul<<<148 * 16, 256>>>((float4*)y, n / 4, nrm, (float4*)x2);
        cudaEventRecord(e0); for (int r = 0; r < 20; ++r) k_mul<<<148 * 16, 256>>>((float4*)y, n / 4, nrm, (float4*)x2);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&t2, e0, e1);
        printf("2^%d: div %.1f us  markstein %.1f us  mismatches %llu of %lld\n", sc, t1 * 50, t2 * 50, tot, n * 7);
        cudaFree(y); cudaFree(x1); cudaFree(x2); cudaFree(nrm); cudaFree(bad);
    }
}
