// kd_common.cuh -- shared device/host helpers for the sm_100a kd-tree build and KNN kernels.
//
// Arithmetic contract (reference core.py:199-228, local_query.py:120-124,
// median.py:143-166): every quantity that decides a split or a neighbour is
// computed in binary64 with explicit round-to-nearest intrinsics (never
// contracted into FMA) in the reference's operation order, so results are
// bit-identical to the CPU reference.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

namespace kdb {

constexpr uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;

// median.py:51-56 _mix64
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = z + GAMMA;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// SplitMix64 output after (j+1) calls of median.py:59-66 _rng_next from `seed`
__host__ __device__ __forceinline__ uint64_t rng_at(uint64_t seed, uint64_t j) {
    uint64_t z = seed + (j + 1) * GAMMA;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// median.py:69-71 _node_seed
__host__ __device__ __forceinline__ uint64_t node_seed(uint64_t seed, uint64_t path, uint64_t salt) {
    return mix64(seed ^ mix64(path) ^ mix64(salt * GAMMA));
}

// order-preserving integer keys; -0.0 is canonicalised to +0.0 so that key
// equality == binary64 equality (the reference compares values, not bits)
__device__ __forceinline__ uint32_t fkey(float v) {
    uint32_t b = __float_as_uint(v);
    if (b == 0x80000000u) b = 0u;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
    uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
    return __uint_as_float(b);
}
__device__ __forceinline__ uint64_t fkey(double v) {
    uint64_t b = (uint64_t)__double_as_longlong(v);
    if (b == 0x8000000000000000ULL) b = 0ULL;
    return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double dkey_inv(uint64_t k) {
    uint64_t b = (k & 0x8000000000000000ULL) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
    return __longlong_as_double((long long)b);
}

template <typename T> struct KeyOf;
template <> struct KeyOf<float> { typedef uint32_t type; static constexpr int bits = 32; };
template <> struct KeyOf<double> { typedef uint64_t type; static constexpr int bits = 64; };
__device__ __forceinline__ float key_inv(uint32_t k, float*) { return fkey_inv(k); }
__device__ __forceinline__ double key_inv(uint64_t k, double*) { return dkey_inv(k); }

// |cum/total - 0.5| exactly as numba evaluates median.py:160
__device__ __forceinline__ double half_diff(int64_t cum, int64_t total) {
    double x = __ddiv_rn((double)cum, (double)total);
    return fabs(__dsub_rn(x, 0.5));
}

struct CudaError {
    std::string msg;
};

}  // namespace kdb

#define KD_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) {                                                          \
            char _b[512];                                                                 \
            snprintf(_b, sizeof(_b), "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), \
                     __FILE__, __LINE__);                                                 \
            throw kdb::CudaError{_b};                                                     \
        }                                                                                 \
    } while (0)
