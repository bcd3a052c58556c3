// lw_common.cuh — shared device helpers for the sm_100a SpMV kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "lw_b200.h"

#define LW_TRY(expr)                                   \
    do {                                               \
        cudaError_t _e = (expr);                       \
        if (_e != cudaSuccess) return (int)_e;         \
    } while (0)

#define LW_LAUNCH_CHECK() LW_TRY(cudaGetLastError())

namespace lw {

constexpr int kWarp = 32;

// Device view of the CSR operand (lw_csr_t with typed pointers).
template <class OffT, class ValT>
struct Csr {
    int64_t rows, cols, nnz;
    const OffT* __restrict__ off;
    const int32_t* __restrict__ col;
    const ValT* __restrict__ val;
};

struct Probe {
    int64_t* lane_atoms;
    int32_t* atom_lane;
    int32_t* atom_tile;
    int32_t* atom_visits;
};

__device__ __forceinline__ void probe_atom(const Probe& p, int64_t atom, int64_t lane,
                                           int64_t tile) {
    if (p.atom_lane) p.atom_lane[atom] = (int32_t)lane;
    if (p.atom_tile) p.atom_tile[atom] = (int32_t)tile;
    if (p.atom_visits) atomicAdd(p.atom_visits + atom, 1);
}

// ---- cache-policy loads --------------------------------------------------
// Loads of read-only operands; LW_VOLATILE_LOADS pins their program order
// (A/B switch: non-volatile lets ptxas hoist/batch them).
#ifdef LW_VOLATILE_LOADS
#define LW_LDASM asm volatile
#else
#define LW_LDASM asm
#endif
// Streaming operands (col_idx, values) are touched once per SpMV: keep them out
// of L1 and mark them evict-first in L2 so the gathered x (reused across rows)
// stays resident in the 126 MB L2 (policy via createpolicy + .L2::cache_hint).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
#ifndef LW_X_POLICY   // A/B: L2 policy of the x gathers (0 evict_last, 1 evict_normal, 2 evict_first, 3 evict_last on 40%)
#define LW_X_POLICY 0
#endif
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    if (LW_X_POLICY == 1) asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    else if (LW_X_POLICY == 2) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else if (LW_X_POLICY == 3) asm("createpolicy.fractional.L2::evict_last.L2::evict_unchanged.b64 %0, 0.4;" : "=l"(p));
    else asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
    int32_t v;
    LW_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(policy_evict_first()));
    return v;
}
__device__ __forceinline__ float ld_stream(const float* p) {
    float v;
    LW_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(v) : "l"(p), "l"(policy_evict_first()));
    return v;
}
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    LW_LDASM("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(policy_evict_first()));
    return v;
}
// Gathered x: read-only path, L1-allocating, evict-last in L2.
#ifndef LW_GATHER_L1
#define LW_GATHER_L1 ""
#endif
__device__ __forceinline__ float ld_gather(const float* p) {
    float v;
    LW_LDASM("ld.global.nc" LW_GATHER_L1 ".L2::cache_hint.f32 %0, [%1], %2;"
                 : "=f"(v) : "l"(p), "l"(policy_evict_last()));
    return v;
}
__device__ __forceinline__ double ld_gather(const double* p) {
    double v;
    LW_LDASM("ld.global.nc" LW_GATHER_L1 ".L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(v) : "l"(p), "l"(policy_evict_last()));
    return v;
}

// Row offsets are read a handful of times per row (search + staging): plain
// read-only loads.
template <class OffT>
__device__ __forceinline__ int64_t ld_off(const OffT* p) {
    return (int64_t)__ldg(p);
}

template <class T>
__device__ __forceinline__ T shfl(T v, int src) {
    return __shfl_sync(0xffffffffu, v, src);
}
template <class T>
__device__ __forceinline__ T shfl_down(T v, int d) {
    return __shfl_down_sync(0xffffffffu, v, d);
}
template <class T>
__device__ __forceinline__ T shfl_up(T v, int d) {
    return __shfl_up_sync(0xffffffffu, v, d);
}

// Warp segmented suffix-reduction from a ballot of segment heads (keys
// nondecreasing across lanes, head = first lane of a run): afterwards the head
// lane of every run holds the run's sum. Each level moves one value (one SHFL
// for fp32 partials, two for fp64); run boundaries come from the head mask.
template <class R>
__device__ __forceinline__ R warp_segsum_heads(R v, int lane, uint32_t heads) {
    // last lane of my run: the lane before the next head above me (or 31)
    const uint32_t above = heads & ~((2u << lane) - 1u);   // heads strictly above lane
    const int seg_end = above ? (__ffs(above) - 2) : (kWarp - 1);
#pragma unroll
    for (int d = 1; d < kWarp; d <<= 1) {
        const R ov = __shfl_down_sync(0xffffffffu, v, d);
        if (lane + d <= seg_end) v += ov;
    }
    return v;
}

// Positions [e0, e1) of one tile of a group_mapped block in the reference's
// member-major order (_fast.py:66-77): member m of M takes block-local positions
// k = m (mod M), so position e0 + i belongs to member (r0 + i) mod M with
// r0 = e0 mod M. Members in ascending order are the offsets
// i = M - r0, ..., rs - 1 (wrapped residues 0, 1, ...), then i = 0, ..., M - r0 - 1
// (residues r0, ..., M - 1), rs = min(e1 - e0, M); each member's positions step
// by M. next() yields them one by one (-1 when done).
struct MemberMajorWalk {
    int64_t e0, e1, M, split, rs, i, k;
    __host__ __device__ MemberMajorWalk(int64_t e0_, int64_t e1_, int64_t M_) : e0(e0_), e1(e1_), M(M_) {
        const int64_t n = e1 - e0;
        rs = n < M ? n : M;
        split = n > 0 ? M - e0 % M : 0;     // offsets >= split are the wrapped residues
        i = split < rs ? split : 0;
        k = n > 0 ? e0 + i : e1;
    }
    __host__ __device__ __forceinline__ int64_t next() {
        if (k >= e1) return -1;
        const int64_t r = k;
        k += M;
        if (k >= e1) {   // this member is done: the next member's first position
            if (i >= split) {                                   // wrapped residues, then offset 0
                i = i + 1 < rs ? i + 1 : 0;                     // (offset 0 exists: split >= 1)
                k = e0 + i;
            } else if (i + 1 < (rs < split ? rs : split)) {
                k = e0 + ++i;
            }                                                   // else k stays >= e1: done
        }
        return r;
    }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Programmatic dependent launch (sm_90+): a kernel launched with launch_pdl may
// start while the previous kernel in the stream is still running — once every
// CTA of that kernel has executed pdl_trigger() or exited. It must call
// pdl_wait() before it reads anything the previous kernel writes. Both are
// no-ops for kernels launched the ordinary way.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

int sm_count();  // cached per device (lw_abi.cu)

}  // namespace lw
