// kd_warp.cuh -- warp-level building blocks for the exact split selection.
//
//  * warp_sort<R>(keys)  : bitonic sort of 32*R keys held striped in registers
//                          (element i = r*32 + lane), shuffles for lane strides,
//                          compile-time register pairs for register strides.
//  * fy_resolve()        : the partial Fisher-Yates draw of median.py:74-85
//                          (m distinct positions of [0,n) from SplitMix64),
//                          computed in parallel: sort (target, step) pairs, then
//                          follow "latest earlier step that targeted this slot"
//                          chains -- bit-identical to the sequential swap loop.
//  * exact warp reductions in binary64 with a fixed butterfly order.
#pragma once
#include "kd_common.cuh"

namespace kdb {

constexpr unsigned FULL = 0xFFFFFFFFu;

template <typename K>
__device__ __forceinline__ K kmin(K a, K b) { return a < b ? a : b; }
template <typename K>
__device__ __forceinline__ K kmax(K a, K b) { return a < b ? b : a; }

template <int JR, int R, typename K>
__device__ __forceinline__ void reg_stage(K (&v)[R], int k, int lane) {
#pragma unroll
    for (int r = 0; r < R; r++) {
        if ((r & JR) == 0 && (r | JR) < R) {
            const int i = r * 32 + lane;
            const bool up = (i & k) == 0;
            K a = v[r], b = v[r | JR];
            if ((a > b) == up) { v[r] = b; v[r | JR] = a; }
        }
    }
}

// ascending bitonic sort of 32*R keys (R a power of two <= 32)
template <int R, typename K>
__device__ __forceinline__ void warp_sort(K (&v)[R]) {
    const int lane = threadIdx.x & 31;
    constexpr int N = R * 32;
    for (int k = 2; k <= N; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j < 32) {
                const bool lower = (lane & j) == 0;
#pragma unroll
                for (int r = 0; r < R; r++) {
                    const int i = r * 32 + lane;
                    const bool up = (i & k) == 0;
                    K o = __shfl_xor_sync(FULL, v[r], j);
                    v[r] = (lower == up) ? kmin(v[r], o) : kmax(v[r], o);
                }
            } else {
                switch (j >> 5) {
                    case 1: reg_stage<1>(v, k, lane); break;
                    case 2: reg_stage<2>(v, k, lane); break;
                    case 4: reg_stage<4>(v, k, lane); break;
                    case 8: reg_stage<8>(v, k, lane); break;
                    case 16: reg_stage<16>(v, k, lane); break;
                    default: break;
                }
            }
        }
    }
}

// element i (runtime) of a striped register array, broadcast to all lanes
template <int R, typename K>
__device__ __forceinline__ K warp_get(const K (&v)[R], int i) {
    K out = 0;
    const int rr = i >> 5, ll = i & 31;
#pragma unroll
    for (int r = 0; r < R; r++) {
        K t = __shfl_sync(FULL, v[r], ll);
        if (r == rr) out = t;
    }
    return out;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = __dadd_rn(x, __shfl_xor_sync(FULL, x, o));
    return x;
}
__device__ __forceinline__ int warp_isum(int x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    return x;
}

// z mod d for d < 2^32 without the 64-bit software division
__device__ __forceinline__ uint64_t mod_u64_u32(uint64_t z, uint32_t d) {
    const uint32_t hi = (uint32_t)(z >> 32), lo = (uint32_t)z;
    const uint64_t x = ((uint64_t)(hi % d) << 32) | lo;  // < d * 2^32
    const double q = floor(__ddiv_rn(__ull2double_rn(x), (double)d));
    int64_t r = (int64_t)(x - (uint64_t)q * (uint64_t)d);
    while (r < 0) r += d;
    while (r >= (int64_t)d) r -= d;
    return (uint64_t)r;
}

// Partial Fisher-Yates (median.py:74-85) resolved in parallel by one warp.
// Writes picked[0..m) (node-relative positions) into shared memory.
// skeys: shared scratch of 32*R entries of type K (K = uint32_t when
// n <= 2^22, else uint64_t); keys are (target << 10) | step.
template <int R, typename K>
__device__ void fy_resolve(uint32_t n, int m, uint64_t seed, K* skeys, uint32_t* picked) {
    const int lane = threadIdx.x & 31;
    K v[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int j = r * 32 + lane;
        if (j < m) {
            const uint64_t z = rng_at(seed, (uint64_t)j);
            const uint32_t tgt = (uint32_t)j + (uint32_t)mod_u64_u32(z, n - (uint32_t)j);
            v[r] = ((K)tgt << 10) | (K)j;
        } else {
            v[r] = ~(K)0;
        }
    }
    warp_sort<R>(v);
#pragma unroll
    for (int r = 0; r < R; r++) skeys[r * 32 + lane] = v[r];
    __syncwarp();
    const int M = R * 32;
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int s = r * 32 + lane;
        const K key = v[r];
        if (key == ~(K)0) continue;
        const uint32_t j = (uint32_t)(key & 1023);
        const uint32_t tgt = (uint32_t)(key >> 10);
        uint32_t val;
        const K prev = s > 0 ? skeys[s - 1] : ~(K)0;
        if (s == 0 || (uint32_t)(prev >> 10) != tgt) {
            val = tgt;  // first step to target this slot: it still holds its own index
        } else {
            // value at slot `tgt` before step j = value that step j' moved there =
            // value at slot j' before step j' (V chain)
            uint32_t t = (uint32_t)(prev & 1023);
            for (;;) {
                const K probe = ((K)t << 10) | (K)t;
                int lo = 0, hi = M;  // lower_bound(probe)
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (skeys[mid] < probe) lo = mid + 1; else hi = mid;
                }
                if (lo > 0 && (uint32_t)(skeys[lo - 1] >> 10) == t) t = (uint32_t)(skeys[lo - 1] & 1023);
                else break;
            }
            val = t;
        }
        picked[j] = val;
    }
    __syncwarp();
}

}  // namespace kdb

namespace kdb {

// ---------------------------------------------------------------------------
// fy_hash: the same partial Fisher-Yates draw as fy_resolve, resolved with a
// shared-memory hash table (target slot -> list of steps that targeted it)
// instead of a sort.  For step j, pred(j) = latest earlier step with the same
// target; V(t) = value at slot t before step t follows the latest step < t that
// targeted t.  Lists are unordered; "latest earlier" is a max over the list.
//   hkey/hhead: FY_HS words each, hnext: m words, out: m words.
// ---------------------------------------------------------------------------
constexpr int FY_HS = 2048;
constexpr uint32_t FY_EMPTY = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t fy_slot0(uint32_t t) { return (t * 0x9E3779B1u) >> (32 - 11); }

__device__ __forceinline__ int fy_find(const uint32_t* hkey, uint32_t t) {
    uint32_t s = fy_slot0(t);
    for (;;) {
        const uint32_t k = hkey[s];
        if (k == t) return (int)s;
        if (k == FY_EMPTY) return -1;
        s = (s + 1) & (FY_HS - 1);
    }
}

// latest step < before in the list of slot s (FY_EMPTY if none)
__device__ __forceinline__ uint32_t fy_latest(const uint32_t* hhead, const uint32_t* hnext, int s, uint32_t before) {
    uint32_t best = FY_EMPTY;
    for (uint32_t x = hhead[s]; x != FY_EMPTY; x = hnext[x])
        if (x < before && (best == FY_EMPTY || x > best)) best = x;
    return best;
}

__device__ __forceinline__ void fy_hash(uint32_t n, int m, uint64_t seed, uint32_t* hkey, uint32_t* hhead, uint32_t* hnext,
                        uint32_t* out) {
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < FY_HS; i += 32) { hkey[i] = FY_EMPTY; hhead[i] = FY_EMPTY; }
    __syncwarp();
    for (int j = lane; j < m; j += 32) {
        const uint64_t z = rng_at(seed, (uint64_t)j);
        const uint32_t t = (uint32_t)j + (uint32_t)mod_u64_u32(z, n - (uint32_t)j);
        uint32_t s = fy_slot0(t);
        for (;;) {
            const uint32_t old = atomicCAS(&hkey[s], FY_EMPTY, t);
            if (old == FY_EMPTY || old == t) break;
            s = (s + 1) & (FY_HS - 1);
        }
        hnext[j] = atomicExch(&hhead[s], (uint32_t)j);
        out[j] = t;
    }
    __syncwarp();
    for (int j = lane; j < m; j += 32) {
        const uint32_t t = out[j];
        uint32_t cur = fy_latest(hhead, hnext, fy_find(hkey, t), (uint32_t)j);
        uint32_t val = t;
        if (cur != FY_EMPTY) {
            for (;;) {  // V(cur): value at slot cur before step cur
                const int s2 = fy_find(hkey, cur);
                const uint32_t p = s2 < 0 ? FY_EMPTY : fy_latest(hhead, hnext, s2, cur);
                if (p == FY_EMPTY) { val = cur; break; }
                cur = p;
            }
        }
        out[j] = val;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// warp_radix_sort: stable LSD radix sort (8-bit digits) of m keys held in
// shared memory (a -> sorted in a; b is scratch of m keys; cnt is 256 words).
// Within a 32-key chunk, equal digits keep lane order via __match_any_sync.
// ---------------------------------------------------------------------------
template <typename K>
__device__ void warp_radix_sort(K* a, K* b, int m, uint32_t* cnt) {
    const int lane = threadIdx.x & 31;
    constexpr int KB = sizeof(K) * 8;
    for (int shift = 0; shift < KB; shift += 8) {
        for (int i = lane; i < 256; i += 32) cnt[i] = 0;
        __syncwarp();
        for (int i = lane; i < m; i += 32) atomicAdd(&cnt[(int)((a[i] >> shift) & 255)], 1u);
        __syncwarp();
        // exclusive scan of the 256 counters (8 per lane)
        uint32_t h[8], s = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) { h[j] = cnt[lane * 8 + j]; s += h[j]; }
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t run = incl - s;
#pragma unroll
        for (int j = 0; j < 8; j++) { cnt[lane * 8 + j] = run; run += h[j]; }
        __syncwarp();
        for (int c = 0; c < m; c += 32) {
            const int i = c + lane;
            const bool v = i < m;
            const K key = v ? a[i] : (K)0;
            const uint32_t dg = v ? (uint32_t)((key >> shift) & 255) : 256u + lane;
            const unsigned peers = __match_any_sync(FULL, dg);
            const int r = __popc(peers & ((1u << lane) - 1));
            const uint32_t base = v ? cnt[dg] : 0;
            __syncwarp();
            if (v) b[base + r] = key;
            if (v && r == 0) cnt[dg] = base + __popc(peers);
            __syncwarp();
        }
        { K* t = a; a = b; b = t; }  // result now in `a` (pointer swap)
        __syncwarp();
    }
    // KB/8 passes: an even number for 32- and 64-bit keys, so the data ends in the caller's `a`
}

}  // namespace kdb
