// kd_warp.cuh -- warp-level building blocks for the exact split selection.
//
//  * warp_sort_t<R>(keys): sorting network on 32*R keys held transposed in
//                          registers (element i = lane*R + r), compile-time
//                          register pairs for strides < R, shuffles above.
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

// compare-exchange: min to a, max to b
template <typename K>
__device__ __forceinline__ void cex(K& a, K& b) {
    const K lo = kmin(a, b), hi = kmax(a, b);
    a = lo;
    b = hi;
}

// Sorting network on 32*R keys held TRANSPOSED in registers: element
// i = lane*R + r.  Flip-bitonic formulation (every comparator ascending, no
// direction bits): merge size KS starts with a flip stage (partner i ^ (KS-1))
// followed by half-cleaners (partner i ^ J).  Strides below R are register
// pairs (2 instructions per pair, compile-time indices); strides >= R are lane
// strides (one shuffle per key).  For R = 32: 40 register stages + 15 shuffle
// stages.
template <int KS, int R, typename K>
__device__ __forceinline__ void flip_stage(K (&v)[R], int lane) {
    if constexpr (KS <= R) {
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int p = r ^ (KS - 1);
            if (r < p) cex(v[r], v[p]);
        }
    } else {
        constexpr int LM = KS / R - 1;  // partner of (lane, r) is (lane ^ LM, R-1-r)
        const bool lower = (lane & (KS / R / 2)) == 0;
#pragma unroll
        for (int r = 0; r < (R + 1) / 2; r++) {
            const int q = R - 1 - r;
            const K a = __shfl_xor_sync(FULL, v[q], LM);  // partner's v[R-1-r]
            if (q != r) {
                const K b = __shfl_xor_sync(FULL, v[r], LM);  // partner's v[r], pairs with my v[q]
                v[q] = lower ? kmin(v[q], b) : kmax(v[q], b);
            }
            v[r] = lower ? kmin(v[r], a) : kmax(v[r], a);
        }
    }
}

template <int J, int R, typename K>
__device__ __forceinline__ void half_stages(K (&v)[R], int lane) {
    if constexpr (J >= 1) {
        if constexpr (J < R) {
#pragma unroll
            for (int r = 0; r < R; r++)
                if ((r & J) == 0) cex(v[r], v[r | J]);
        } else {
            constexpr int LM = J / R;
            const bool lower = (lane & LM) == 0;
#pragma unroll
            for (int r = 0; r < R; r++) {
                const K o = __shfl_xor_sync(FULL, v[r], LM);
                v[r] = lower ? kmin(v[r], o) : kmax(v[r], o);
            }
        }
        half_stages<J / 2, R>(v, lane);
    }
}

template <int KS, int N, int R, typename K>
__device__ __forceinline__ void merges(K (&v)[R], int lane) {
    if constexpr (KS <= N) {
        flip_stage<KS, R>(v, lane);
        half_stages<KS / 4, R>(v, lane);
        merges<KS * 2, N, R>(v, lane);
    }
}

// ascending sort of 32*R keys (R a power of two <= 32); result transposed:
// sorted element s sits in lane s / R, register s % R
template <int R, typename K>
__device__ __forceinline__ void warp_sort_t(K (&v)[R]) {
    merges<2, 32 * R, R>(v, threadIdx.x & 31);
}

// The same network with the cross-lane merges rolled: every merge of more than R keys is
// [lane flip] [lane half-cleaners, stride ks/4 .. 1 lanes] [register half-cleaners R/2 .. 1],
// identical code for every merge size, so it runs as a loop over the merge size with runtime
// shuffle masks.  Same comparators, same result; the instruction stream is ~5x shorter, which
// matters where the kernel is bound by instruction fetch (straight-line code is fetched, not
// reused: k_subtree's split functions, k_sample's 1024-key sorts).
template <int R, typename K>
__device__ __forceinline__ void warp_sort_rolled(K (&v)[R]) {
    const int lane = threadIdx.x & 31;
    merges<2, R, R>(v, lane);  // each lane's R keys, in registers
#pragma unroll 1
    for (int ks = 2; ks <= 32; ks <<= 1) {  // lanes per merged run
        {
            const int lm = ks - 1;  // partner of (lane, r) is (lane ^ lm, R-1-r)
            const bool lower = (lane & (ks >> 1)) == 0;
#pragma unroll
            for (int r = 0; r < (R + 1) / 2; r++) {
                const int q = R - 1 - r;
                const K a = __shfl_xor_sync(FULL, v[q], lm);
                if (q != r) {
                    const K b = __shfl_xor_sync(FULL, v[r], lm);
                    v[q] = lower ? kmin(v[q], b) : kmax(v[q], b);
                }
                v[r] = lower ? kmin(v[r], a) : kmax(v[r], a);
            }
        }
#pragma unroll 1
        for (int jl = ks >> 2; jl >= 1; jl >>= 1) {
            const bool lower = (lane & jl) == 0;
#pragma unroll
            for (int r = 0; r < R; r++) {
                const K o = __shfl_xor_sync(FULL, v[r], jl);
                v[r] = lower ? kmin(v[r], o) : kmax(v[r], o);
            }
        }
        half_stages<R / 2, R>(v, lane);
    }
}

// the sorted element before (lane, r) in a transposed sorted array; `up` is
// __shfl_up_sync(v[R-1], 1) (the previous lane's last key), `none` for element 0
template <int R, typename K>
__device__ __forceinline__ K sorted_prev(const K (&v)[R], int r, int lane, K up, K none) {
    return r > 0 ? v[r > 0 ? r - 1 : 0] : (lane > 0 ? up : none);
}

// bank-conflict-free shared-memory slot of logical index s (bijection on each 32-word row)
__device__ __forceinline__ int swz(int s) { return s ^ ((s >> 5) & 31); }

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
// gidx (optional, 32*R u16): per slot t < 32*R, sorted index of the first step
// that targets t -- turns each chain hop into one or two shared loads instead of
// a binary search.
template <int R, typename K>
__device__ __noinline__ void fy_resolve(uint32_t n, int m, uint64_t seed, K* skeys, uint32_t* picked, uint16_t* gidx = nullptr) {
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
    warp_sort_t<R>(v);
#pragma unroll
    for (int r = 0; r < R; r++) skeys[swz(lane * R + r)] = v[r];
    const int M = R * 32;
    const K up = __shfl_up_sync(FULL, v[R - 1], 1);
    if (gidx) {
        for (int i = lane; i < M; i += 32) gidx[i] = 0xFFFF;
        __syncwarp();
#pragma unroll
        for (int r = 0; r < R; r++) {
            const K prev = sorted_prev<R>(v, r, lane, up, ~(K)0);
            const uint32_t tgt = (uint32_t)(v[r] >> 10);
            if (v[r] != ~(K)0 && tgt < (uint32_t)M && (lane * R + r == 0 || (uint32_t)(prev >> 10) != tgt))
                gidx[tgt] = (uint16_t)(lane * R + r);
        }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; r++) {
        const int s = lane * R + r;
        const K key = v[r];
        const K prev = sorted_prev<R>(v, r, lane, up, ~(K)0);
        if (key == ~(K)0) continue;
        const uint32_t j = (uint32_t)(key & 1023);
        const uint32_t tgt = (uint32_t)(key >> 10);
        uint32_t val;
        if (s == 0 || (uint32_t)(prev >> 10) != tgt) {
            val = tgt;  // first step to target this slot: it still holds its own index
        } else {
            // value at slot `tgt` before step j = value that step j' moved there =
            // value at slot j' before step j' (V chain)
            uint32_t t = (uint32_t)(prev & 1023);
            if (gidx) {
                for (;;) {  // latest step < t that targeted slot t (its group is sorted by step)
                    int g = gidx[t];
                    if (g == 0xFFFF) break;
                    uint32_t best = 0xFFFFFFFFu;
                    for (; g < M; g++) {
                        const K gk = skeys[swz(g)];
                        if ((uint32_t)(gk >> 10) != t || (uint32_t)(gk & 1023) >= t) break;
                        best = (uint32_t)(gk & 1023);
                    }
                    if (best == 0xFFFFFFFFu) break;
                    t = best;
                }
            } else for (;;) {
                const K probe = ((K)t << 10) | (K)t;
                int lo = 0, hi = M;  // lower_bound(probe)
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (skeys[swz(mid)] < probe) lo = mid + 1; else hi = mid;
                }
                if (lo > 0) {
                    const K pk = skeys[swz(lo - 1)];
                    if ((uint32_t)(pk >> 10) == t) { t = (uint32_t)(pk & 1023); continue; }
                }
                break;
            }
            val = t;
        }
        picked[j] = val;
    }
    __syncwarp();
}

// Partial Fisher-Yates for nodes of at most FYD_MAX points, without sorting.
// Same draws as fy_resolve (median.py:74-85).  Step j targets r_j in [j, n);
// the value drawn is the one at slot r_j before step j.  A slot s >= j is only
// ever written by earlier steps that targeted it, so with
//   prev(j) = latest step i < j with r_i = r_j        (none -> slot untouched)
//   back(t) = latest step i < t with r_i = t, t < m   (none -> slot t untouched)
//   W(i)    = value at slot i before step i = back(i) ? W(back(i)) : i
// the draw is picked[j] = prev(j) ? W(prev(j)) : r_j.  prev() comes from 32
// rounds of 32 steps against a direct table last[slot] (latest step so far),
// with same-round collisions resolved by __match_any_sync; back(t) is prev(t)
// when step t targeted itself, else the final last[t] (no step after t can
// target t).  Shared scratch: last[n] u16, back[m] u16, picked[m] u32.
constexpr int FYD_MAX = 4096;
constexpr uint16_t FYD_NONE = 0xFFFF;

template <int R>
__device__ __noinline__ void fy_direct(uint32_t n, int m, uint64_t seed, uint16_t* last, uint16_t* back, uint32_t* picked) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1;
    for (uint32_t i = lane; i < (n + 1) / 2; i += 32) reinterpret_cast<uint32_t*>(last)[i] = 0xFFFFFFFFu;
    __syncwarp();
#pragma unroll 1
    for (int r = 0; r < R; r++) {
        const int j = r * 32 + lane;
        const bool act = j < m;
        uint32_t tgt = 0xFFFFFFFFu;
        if (act) {
            const uint64_t z = rng_at(seed, (uint64_t)j);
            tgt = (uint32_t)j + (uint32_t)mod_u64_u32(z, n - (uint32_t)j);
        }
        const unsigned grp = __match_any_sync(FULL, tgt);
        const unsigned lower = grp & lt;
        uint32_t pv = FYD_NONE;
        if (act) pv = lower ? (uint32_t)(r * 32 + 31 - __clz(lower)) : (uint32_t)last[tgt];
        __syncwarp();
        // the highest lane of each target group records the latest step
        if (act && (grp >> lane) == 1u) last[tgt] = (uint16_t)j;
        if (act) picked[j] = tgt | (pv << 16);
        __syncwarp();
    }
    for (int j = lane; j < m; j += 32) {
        const uint32_t w = picked[j];
        const uint32_t tgt = w & 0xFFFFu;
        back[j] = tgt == (uint32_t)j ? (uint16_t)(w >> 16) : last[j];
    }
    __syncwarp();
    for (int j = lane; j < m; j += 32) {
        const uint32_t w = picked[j];
        uint32_t i = w >> 16;
        uint32_t val = w & 0xFFFFu;
        if (i != FYD_NONE) {
            while (back[i] != FYD_NONE) i = back[i];
            val = i;
        }
        picked[j] = val;
    }
    __syncwarp();
}

// Partial Fisher-Yates for nodes of FYD_MAX < n <= 2^22 points: the algorithm of
// fy_direct with the last[] table replaced by an open-addressing hash table of
// FYH_SLOTS entries (target << 10 | latest step) -- at most m <= 1024 distinct
// targets are ever recorded, so the table is at most half full and needs no
// sorting of the draws (fy_resolve) whatever the node size.
//   lookup  by the lowest lane of every same-target group of a 32-step round
//           (the other lanes' previous step is the next lower lane of the group);
//   insert  by the same lane, after every lookup of the round has finished:
//           the group's highest step overwrites the target's entry, or claims
//           the free slot that ended the probe (atomicCAS against other groups).
// Shared scratch: tab[FYH_SLOTS] u32, back[m] u16, picked[m] u32.
constexpr int FYH_SLOTS = 2048;
constexpr uint32_t FYH_EMPTY = 0xFFFFFFFFu;
constexpr uint32_t FYH_NONE = 1023u;  // a previous step is < 1023

__device__ __forceinline__ uint32_t fyh_slot(uint32_t tgt) { return (tgt * 2654435761u) >> 21; }

// entry of `tgt`: returns the step recorded for it (FYH_NONE if absent); h = its slot or the free slot that ended the probe
__device__ __forceinline__ uint32_t fyh_find(const uint32_t* tab, uint32_t tgt, uint32_t& h) {
    h = fyh_slot(tgt);
    for (;;) {
        const uint32_t e = tab[h];
        if (e == FYH_EMPTY) return FYH_NONE;
        if ((e >> 10) == tgt) return e & 1023u;
        h = (h + 1) & (FYH_SLOTS - 1);
    }
}

template <int R>
__device__ __noinline__ void fy_hash(uint32_t n, int m, uint64_t seed, uint32_t* tab, uint16_t* back, uint32_t* picked) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1;
    for (int i = lane; i < FYH_SLOTS; i += 32) tab[i] = FYH_EMPTY;
    __syncwarp();
#pragma unroll 1
    for (int r = 0; r < R; r++) {
        const int j = r * 32 + lane;
        const bool act = j < m;
        uint32_t tgt = 0xFFFFFFFFu;
        if (act) {
            const uint64_t z = rng_at(seed, (uint64_t)j);
            tgt = (uint32_t)j + (uint32_t)mod_u64_u32(z, n - (uint32_t)j);
        }
        const unsigned grp = __match_any_sync(FULL, tgt);
        const unsigned lower = grp & lt;
        uint32_t pv = FYH_NONE, h = 0;
        if (act) {
            if (lower) pv = (uint32_t)(r * 32 + 31 - __clz(lower));
            else pv = fyh_find(tab, tgt, h);
        }
        __syncwarp();
        if (act && !lower) {
            const uint32_t val = (tgt << 10) | (uint32_t)(r * 32 + 31 - __clz(grp));
            if (pv != FYH_NONE) {
                tab[h] = val;  // the target's own entry: no other group writes it
            } else {
                for (;;) {  // claim a free slot (other groups may race for the same one)
                    const uint32_t old = atomicCAS(&tab[h], FYH_EMPTY, val);
                    if (old == FYH_EMPTY) break;
                    h = (h + 1) & (FYH_SLOTS - 1);
                }
            }
        }
        if (act) picked[j] = tgt | (pv << 22);
        __syncwarp();
    }
    // back(t) = latest step i < t that targeted slot t: step t's own previous step if it
    // targeted itself, else the final entry of t (no later step can target t)
    for (int j = lane; j < m; j += 32) {
        const uint32_t w = picked[j];
        uint32_t h;
        const uint32_t b = (w & 0x3FFFFFu) == (uint32_t)j ? (w >> 22) : fyh_find(tab, (uint32_t)j, h);
        back[j] = (uint16_t)b;
    }
    __syncwarp();
    for (int j = lane; j < m; j += 32) {
        const uint32_t w = picked[j];
        uint32_t i = w >> 22;
        uint32_t val = w & 0x3FFFFFu;
        if (i != FYH_NONE) {
            while (back[i] != FYH_NONE) i = back[i];
            val = i;
        }
        picked[j] = val;
    }
    __syncwarp();
}

}  // namespace kdb
