/*
 * lw_hash.h — counter-based hashing shared by the device generators
 * (paper_2301_04792_b200/csrc/generators.cu), the host oracle (oracle/lw_oracle.c)
 * and the NumPy restatement used by the CPU tests. Every synthetic input this
 * project builds beyond the reference's own NumPy generators (R-MAT, banded
 * values) is a pure function of (seed, counter), so the CPU and the GPU produce
 * bit-identical CSR matrices without sharing an RNG stream.
 */
#ifndef LW_HASH_H
#define LW_HASH_H

#include <stdint.h>

#if defined(__CUDACC__)
#define LW_HD __host__ __device__ __forceinline__
#else
#define LW_HD static inline
#endif

#define LW_GOLDEN 0x9E3779B97F4A7C15ULL

/* splitmix64 finalizer */
LW_HD uint64_t lw_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* per-edge stream root */
LW_HD uint64_t lw_edge_root(uint64_t seed, uint64_t edge) {
    return lw_mix64(lw_mix64(seed + LW_GOLDEN) ^ (edge * 0xD6E8FEB86659FD93ULL));
}

/* 32 random bits for R-MAT level `level` (0 = most significant bit) of an edge */
LW_HD uint32_t lw_level_bits(uint64_t root, int level) {
    uint64_t w = lw_mix64(root + (uint64_t)(level / 2 + 1) * LW_GOLDEN);
    return (level & 1) ? (uint32_t)(w >> 32) : (uint32_t)w;
}

/* R-MAT key (row << scale | col) of one edge */
LW_HD uint64_t lw_rmat_key(uint64_t seed, uint64_t edge, int scale, uint32_t t_a,
                           uint32_t t_ab, uint32_t t_abc) {
    uint64_t root = lw_edge_root(seed, edge);
    uint64_t row = 0, col = 0;
    for (int level = 0; level < scale; ++level) {
        uint32_t r = lw_level_bits(root, level);
        uint64_t rb = (r >= t_ab) ? 1u : 0u;                 /* quadrants c, d */
        uint64_t cb = ((r >= t_a && r < t_ab) || r >= t_abc) ? 1u : 0u; /* b, d */
        row = (row << 1) | rb;
        col = (col << 1) | cb;
    }
    return (row << scale) | col;
}

/* Uniform position in [0, space) of draw i (the C2u / C4-uniform generator):
 * the high 64 bits of a 64x64-bit product of the draw's root with space. */
LW_HD uint64_t lw_uniform_key(uint64_t seed, uint64_t i, uint64_t space) {
    const uint64_t r = lw_edge_root(seed ^ 0x2545F4914F6CDD1DULL, i);
#ifdef __CUDA_ARCH__
    return __umul64hi(r, space);
#else
    return (uint64_t)(((unsigned __int128)r * space) >> 64);
#endif
}

/* U[-1, 1) value keyed by a 64-bit position */
LW_HD double lw_hash_value(uint64_t seed, uint64_t key) {
    uint64_t h = lw_mix64(lw_mix64(seed ^ 0x5851F42D4C957F2DULL) + key * LW_GOLDEN);
    return (double)(h >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}

#endif /* LW_HASH_H */
