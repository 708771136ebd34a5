// kd_build.cuh -- reference-exact kd-tree construction on sm_100a (compiled once per
// coordinate type by kd_build_f32.cu / kd_build_f64.cu).
//
// Reproduces kdknn.local_tree.build_local_tree (local_tree.py:436-574) byte for
// byte: same split dimension (max sample variance, local_tree.py:111-146), same
// split value (sampled-histogram approximate median with exact fallback,
// local_tree.py:147-180 + median.py:74-166), same stable partition
// (local_tree.py:183-206), same canonical preorder numbering
// (local_tree.py:320-374) and the same packed bucket order (pack_buckets,
// local_tree.py:402-405).
//
// GPU structure:
//   breadth-first levels for nodes larger than the sample size (global memory,
//   SoA coordinates ping-ponged between two buffers):
//     k_sample   warp/node  exact Fisher-Yates draws (direct / hash table), certified
//                           variance order, sorted unique median sample, 128-boundary window
//     k_hist     tile/CTA   windowed full-data histogram of the split dim
//     k_select   warp/node  exact binary64 median selection from the window
//     k_slow     CTA/node   exact slow path (full histogram, exact fallback,
//                           next dimensions) -- only for flagged nodes
//     k_tile_left/scan/k_scatter_tma (k_scatter for D > 3)  stable segmented partition of
//                           coords + row ids, TMA-fed (per-half-tile left counts from
//                           k_hist's window rows)
//     k_children thread/node child records, next level, subtree tasks
//   then one CTA (two warps) per subtree of <= min(1024, samples) points, built entirely
//   in shared memory (k_subtree), and a preorder stitch (k_top_* / k_relocate).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <vector>

#include "kd_arena.cuh"
#include "kd_common.cuh"
#include "kd_tree.cuh"
#include "kd_warp.cuh"

namespace kdb {

constexpr int MAXS = 1024;       // max sample size supported on device
constexpr int WIN = 128;         // histogram window (boundaries around the sample median; +-4 sigma of its rank)
constexpr int TILE = 4096;       // elements per tile CTA
constexpr int TILE_THREADS = 256;
constexpr int SUB = 2;  // partition half-tiles per tile (k_scatter moves one per CTA)
constexpr int SAMPLE_WARPS = 4;
constexpr int SLOW_THREADS = 256;
constexpr double U64 = 1.1102230246251565e-16;  // 2^-53

enum { ST_SAMPLED = 0, ST_SLOW = 1, ST_LEAF = 2, ST_SPLIT = 3 };
enum { TS_INTERIOR = 0, TS_TASK = 1 };

struct LNode {
    int64_t start;
    int32_t n;
    int32_t depth;
    uint64_t path;
    int32_t slot;
    uint32_t tile_off;
};

struct Split {
    int32_t status;
    int32_t dim;
    int32_t nb;
    int32_t wlo;
    int32_t whi;
    int32_t wsel;  // window index of the chosen split value (k_select), -1 when the slow path chose it
    double value;
    int64_t nl;
    unsigned long long L;
};

struct Task {
    int64_t start;
    int32_t n;
    int32_t depth;
    uint64_t path;
    int32_t slot;
    int32_t src;   // which coordinate buffer holds the points
    int32_t leaf;  // degenerate leaf (all dimensions constant)
    int32_t pad;
};

struct DevCtx {
    int dims;
    int64_t N;
    int64_t bucket, ms, vs;
    uint64_t seed;
    int ts;  // subtree threshold
};

template <typename T>
__device__ __forceinline__ typename KeyOf<T>::type tkey(T v) { return fkey(v); }

// ----------------------------------------------------------------------------
// certified max-variance dimension (local_tree.py:111-146)
// fast path: binary64 warp-tree sums with a rigorous bound on the difference to
// the reference's sequential sums; if the winner is not separated from every
// other candidate by the bound, the caller recomputes sequentially.
// ----------------------------------------------------------------------------
__device__ __forceinline__ double ssd_bound(double s2, double sabs, int t) {
    const double tt = (double)t;
    const double am = sabs / tt;
    const double dm = (tt + 2.0) * U64 * am;
    return 4.0 * (tt + 4.0) * U64 * s2 + 2.0 * tt * dm * dm + 1e-300;
}

// ============================================================================
// k_sample: one warp per breadth-first node
// ============================================================================
template <typename T, int DT, bool BIG>
__global__ void __launch_bounds__(SAMPLE_WARPS * 32)
k_sample(const T* __restrict__ src, const LNode* __restrict__ nodes, int K, DevCtx c, Split* split,
         T* __restrict__ wb, uint32_t* __restrict__ wf) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int DC = DT > 0 ? DT : 16;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ni = blockIdx.x * SAMPLE_WARPS + warp;
    if (ni >= K) return;
    const LNode nd = nodes[ni];
    const uint32_t n = (uint32_t)nd.n;
    // nodes above 2^22 points need 64-bit (target, step) keys; they are few and
    // get their own instantiation so the common one stays small
    if (BIG != (n > (1u << 22))) return;
    typedef typename std::conditional<BIG, uint64_t, uint32_t>::type FK;
    // per warp: region 0 = FY sort keys (MAXS FK) or the direct table (FYD_MAX u16),
    // then picked (MAXS u32), then gidx / back (MAXS u16)
    constexpr size_t R0 = sizeof(FK) * MAXS > 2 * FYD_MAX ? sizeof(FK) * MAXS : 2 * FYD_MAX;
    FK* skeys = reinterpret_cast<FK*>(smem_raw + warp * R0);
    uint16_t* dlast = reinterpret_cast<uint16_t*>(skeys);
    uint32_t* picked = reinterpret_cast<uint32_t*>(smem_raw + SAMPLE_WARPS * R0) + warp * MAXS;
    uint16_t* gidx = reinterpret_cast<uint16_t*>(smem_raw + SAMPLE_WARPS * (R0 + 4 * MAXS)) + warp * MAXS;
    const bool direct = !BIG && n <= (uint32_t)FYD_MAX;
    const int D = DT > 0 ? DT : c.dims;
    const int64_t N = c.N;

    // --- variance sample (local_tree.py:122-132)
    const int take = (int)min((int64_t)n, c.vs);
    const uint64_t vseed = node_seed(c.seed, nd.path, 0);
    if (direct) fy_direct<32>(n, take, vseed, dlast, gidx, picked);
    else if constexpr (!BIG) fy_hash<32>(n, take, vseed, reinterpret_cast<uint32_t*>(skeys), gidx, picked);
    else fy_resolve<32, FK>(n, take, vseed, skeys, picked, gidx);

    int d0 = 0;
    double b0 = 0.0, e0 = 0.0;
    double s2v[DC], eb[DC];
#pragma unroll
    for (int d = 0; d < DC; d++) {
        s2v[d] = 0.0;
        eb[d] = 0.0;
        if (d >= D) continue;
        const T* row = src + (int64_t)d * N + nd.start;
        // every gather of this dimension in flight at once; both passes read the registers
        T xs[MAXS / 32];
#pragma unroll
        for (int r = 0; r < MAXS / 32; r++) {
            const int j = r * 32 + lane;
            xs[r] = j < take ? row[picked[j]] : T(0);
        }
        double s1 = 0.0, sa = 0.0;
#pragma unroll
        for (int r = 0; r < MAXS / 32; r++) {
            if (r * 32 + lane < take) {
                const double x = (double)xs[r];
                s1 = __dadd_rn(s1, x);
                sa = __dadd_rn(sa, fabs(x));
            }
        }
        s1 = warp_sum(s1);
        sa = warp_sum(sa);
        const double mean = __ddiv_rn(s1, (double)take);
        double s2 = 0.0;
#pragma unroll
        for (int r = 0; r < MAXS / 32; r++) {
            if (r * 32 + lane < take) {
                const double df = __dsub_rn((double)xs[r], mean);
                s2 = __dadd_rn(s2, __dmul_rn(df, df));
            }
        }
        s2v[d] = warp_sum(s2);
        eb[d] = ssd_bound(s2v[d], sa, take);
        if (d == 0 || s2v[d] > b0) { d0 = d; b0 = s2v[d]; e0 = eb[d]; }
    }
    bool certified = true;
#pragma unroll
    for (int d = 0; d < DC; d++)
        if (d < D && d != d0 && !(b0 - s2v[d] > e0 + eb[d])) certified = false;
    if (!certified) {
        // exact sequential recomputation in draw order (rare: near-ties)
        double exact = 0.0;
        if (lane < D) {
            const T* row = src + (int64_t)lane * N + nd.start;
            double mean = 0.0;
            for (int j = 0; j < take; j++) mean = __dadd_rn(mean, (double)row[picked[j]]);
            mean = __ddiv_rn(mean, (double)take);
            double s = 0.0;
            for (int j = 0; j < take; j++) {
                const double df = __dsub_rn((double)row[picked[j]], mean);
                s = __dadd_rn(s, __dmul_rn(df, df));
            }
            exact = s;
        }
        d0 = 0;
        double best = __shfl_sync(FULL, exact, 0);
        for (int d = 1; d < D; d++) {
            const double e = __shfl_sync(FULL, exact, d);
            if (-e < -best) { best = e; d0 = d; }  // np.argsort(-ssd, mergesort)[0]
        }
    }

    // --- median sample of dim d0 (local_tree.py:149-156)
    const int m = (int)min((int64_t)n, c.ms);
    const uint64_t mseed = node_seed(c.seed, nd.path, 1ULL + (uint64_t)d0);
    __syncwarp();
    if (direct) fy_direct<32>(n, m, mseed, dlast, gidx, picked);
    else if constexpr (!BIG) fy_hash<32>(n, m, mseed, reinterpret_cast<uint32_t*>(skeys), gidx, picked);
    else fy_resolve<32, FK>(n, m, mseed, skeys, picked, gidx);
    typedef typename KeyOf<T>::type Key;
    const T* row = src + (int64_t)d0 * N + nd.start;
    Key kv[32];
#pragma unroll
    for (int r = 0; r < 32; r++) {
        const int j = r * 32 + lane;
        kv[r] = j < m ? tkey(row[picked[j]]) : ~(Key)0;
    }
    warp_sort_rolled<32>(kv);  // rolled cross-lane merges: -0.65 ms over the 7 k_sample levels of C3
    // np.unique: first element of each run of equal keys; boundary index = rank of run.
    // Sorted element s = lane*32 + r.
    const int mid = m / 2;
    const Key kup = __shfl_up_sync(FULL, kv[31], 1);
    unsigned fmask = 0;  // bit r: element (lane, r) starts a run
    int cle_l = 0;
#pragma unroll
    for (int r = 0; r < 32; r++) {
        const int s = lane * 32 + r;
        const Key prev = sorted_prev<32>(kv, r, lane, kup, kv[0]);
        const bool first = s < m && (s == 0 || kv[r] != prev);
        fmask |= (unsigned)first << r;
        cle_l += first && s <= mid;  // runs starting at or before sorted position `mid`
    }
    const int nf = __popc(fmask);
    int incl = nf;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    const int nb = __shfl_sync(FULL, incl, 31);
    const int cle = warp_isum(cle_l);
    const int center = cle - 1;
    int wlo = max(0, center - WIN / 2);
    const int whi = min(nb, wlo + WIN);
    wlo = max(0, whi - WIN);
    Split* sp = split + ni;
    T* wbn = wb + (int64_t)ni * WIN;
    {
        int bi = incl - nf;  // runs before this lane
#pragma unroll
        for (int r = 0; r < 32; r++) {
            if ((fmask >> r) & 1u) {
                if (bi >= wlo && bi < whi) wbn[bi - wlo] = key_inv(kv[r], (T*)nullptr);
                bi++;
            }
        }
    }
    uint32_t* wfn = wf + (int64_t)ni * WIN;
    for (int i = lane; i < WIN; i += 32) wfn[i] = 0;
    if (lane == 0) {
        sp->status = ST_SAMPLED;
        sp->dim = d0;
        sp->nb = nb;
        sp->wlo = wlo;
        sp->whi = whi;
        sp->value = 0.0;
        sp->nl = 0;
        sp->L = 0ULL;
    }
}

// ============================================================================
// k_sample_cta: the same split choice as k_sample with one 1024-thread CTA per
// node (one sample element per thread) -- for the shallow levels, where a
// level has too few nodes to fill the GPU with warps and a warp per node is
// latency bound (gathers from a node spanning up to the whole point set).
// ============================================================================
constexpr int CTA_S = 1024;

// ascending sort of one key per thread over the block (flip-bitonic network;
// strides < 32 by shuffles, larger ones through two ping-pong shared buffers,
// one barrier per shared stage).  Returns the buffer holding the sorted keys.
template <typename K>
__device__ K* block_sort(K key, K* a, K* b) {
    const int tid = threadIdx.x;
    K* buf[2] = {a, b};
    int pb = 0;
    for (int ks = 2; ks <= CTA_S; ks <<= 1) {
        for (int j = ks >> 1; j > 0; j >>= 1) {
            const int pm = j == (ks >> 1) ? ks - 1 : j;  // flip stage first, then half-cleaners
            const bool lower = (tid & j) == 0;
            K o;
            if (pm < 32) {
                o = __shfl_xor_sync(FULL, key, pm);
            } else {
                buf[pb][tid] = key;
                __syncthreads();
                o = buf[pb][tid ^ pm];
                pb ^= 1;
            }
            key = lower ? kmin(key, o) : kmax(key, o);
        }
    }
    buf[pb][tid] = key;
    __syncthreads();
    return buf[pb];
}

// partial Fisher-Yates (median.py:74-85) with one step per thread: sort the
// (target, step) keys, then resolve "latest earlier step on this slot" chains.
template <typename FK>
__device__ void cta_fy(uint32_t n, int m, uint64_t seed, FK* ka, FK* kb, uint32_t* picked, uint16_t* gidx) {
    const int tid = threadIdx.x;
    FK key = ~(FK)0;
    if (tid < m) {
        const uint64_t z = rng_at(seed, (uint64_t)tid);
        const uint32_t tgt = (uint32_t)tid + (uint32_t)mod_u64_u32(z, n - (uint32_t)tid);
        key = ((FK)tgt << 10) | (FK)tid;
    }
    const FK* sk = block_sort<FK>(key, ka, kb);
    const FK k = sk[tid];
    const FK prev = tid > 0 ? sk[tid - 1] : ~(FK)0;
    const uint32_t tgt = (uint32_t)(k >> 10);
    // gidx[t]: sorted index of the first step that targets slot t < CTA_S
    gidx[tid] = 0xFFFF;
    __syncthreads();
    if (k != ~(FK)0 && tgt < (uint32_t)CTA_S && (tid == 0 || (uint32_t)(prev >> 10) != tgt)) gidx[tgt] = (uint16_t)tid;
    __syncthreads();
    if (k != ~(FK)0) {
        const uint32_t j = (uint32_t)(k & 1023);
        uint32_t val = tgt;
        if (tid > 0 && (uint32_t)(prev >> 10) == tgt) {
            uint32_t t = (uint32_t)(prev & 1023);
            for (;;) {  // latest step < t that targeted slot t
                int g = gidx[t];
                if (g == 0xFFFF) break;
                uint32_t best = 0xFFFFFFFFu;
                for (; g < CTA_S; g++) {
                    const FK gk = sk[g];
                    if ((uint32_t)(gk >> 10) != t || (uint32_t)(gk & 1023) >= t) break;
                    best = (uint32_t)(gk & 1023);
                }
                if (best == 0xFFFFFFFFu) break;
                t = best;
            }
            val = t;
        }
        picked[j] = val;
    }
    __syncthreads();
}

// binary64 block sum (fixed tree order; every warp reduces the partials itself)
__device__ __forceinline__ double block_sum(double x, double* red) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    x = warp_sum(x);
    if (lane == 0) red[warp] = x;
    __syncthreads();
    const double y = warp_sum(red[lane]);
    __syncthreads();
    return y;
}

template <typename T, int DT>
__global__ void __launch_bounds__(CTA_S, 1)
k_sample_cta(const T* __restrict__ src, const LNode* __restrict__ nodes, DevCtx c, Split* split,
             T* __restrict__ wb, uint32_t* __restrict__ wf) {
    __shared__ uint64_t ka[CTA_S], kb[CTA_S];
    __shared__ uint32_t picked[CTA_S];
    __shared__ uint16_t gidx[CTA_S];
    __shared__ double red[32];
    __shared__ double s_s2[16], s_eb[16];
    __shared__ int ired[32];
    __shared__ int s_cle;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int ni = blockIdx.x;
    const LNode nd = nodes[ni];
    const uint32_t n = (uint32_t)nd.n;
    const bool big = n > (1u << 22);
    const int D = DT > 0 ? DT : c.dims;
    const int64_t N = c.N;

    // --- variance sample (local_tree.py:122-132)
    const int take = (int)min((int64_t)n, c.vs);
    const uint64_t vseed = node_seed(c.seed, nd.path, 0);
    if (big) cta_fy<uint64_t>(n, take, vseed, ka, kb, picked, gidx);
    else cta_fy<uint32_t>(n, take, vseed, reinterpret_cast<uint32_t*>(ka), reinterpret_cast<uint32_t*>(kb), picked, gidx);
    const bool act = tid < take;
    const uint32_t pj = act ? picked[tid] : 0u;
    int d0 = 0;
    double b0 = 0.0, e0 = 0.0;
    for (int d = 0; d < D; d++) {
        const T* row = src + (int64_t)d * N + nd.start;
        const double x = act ? (double)row[pj] : 0.0;
        const double s1 = block_sum(x, red);
        const double sa = block_sum(fabs(x), red);
        const double mean = __ddiv_rn(s1, (double)take);
        const double df = act ? __dsub_rn(x, mean) : 0.0;
        const double s2 = block_sum(__dmul_rn(df, df), red);
        const double eb = ssd_bound(s2, sa, take);
        if (tid == 0) { s_s2[d] = s2; s_eb[d] = eb; }
        if (d == 0 || s2 > b0) { d0 = d; b0 = s2; e0 = eb; }
    }
    __syncthreads();
    bool certified = true;
    for (int d = 0; d < D; d++)
        if (d != d0 && !(b0 - s_s2[d] > e0 + s_eb[d])) certified = false;
    if (!certified) {
        // exact sequential recomputation in draw order (rare: near-ties)
        if (tid < D) {
            const T* row = src + (int64_t)tid * N + nd.start;
            double mean = 0.0;
            for (int j = 0; j < take; j++) mean = __dadd_rn(mean, (double)row[picked[j]]);
            mean = __ddiv_rn(mean, (double)take);
            double s = 0.0;
            for (int j = 0; j < take; j++) {
                const double df = __dsub_rn((double)row[picked[j]], mean);
                s = __dadd_rn(s, __dmul_rn(df, df));
            }
            red[tid] = s;
        }
        __syncthreads();
        d0 = 0;
        double best = red[0];
        for (int d = 1; d < D; d++) {
            const double e = red[d];
            if (-e < -best) { best = e; d0 = d; }  // np.argsort(-ssd, mergesort)[0]
        }
    }
    __syncthreads();

    // --- median sample of dim d0 (local_tree.py:149-156)
    const int m = (int)min((int64_t)n, c.ms);
    const uint64_t mseed = node_seed(c.seed, nd.path, 1ULL + (uint64_t)d0);
    if (big) cta_fy<uint64_t>(n, m, mseed, ka, kb, picked, gidx);
    else cta_fy<uint32_t>(n, m, mseed, reinterpret_cast<uint32_t*>(ka), reinterpret_cast<uint32_t*>(kb), picked, gidx);
    typedef typename KeyOf<T>::type Key;
    const T* row = src + (int64_t)d0 * N + nd.start;
    const Key key = tid < m ? tkey(row[picked[tid]]) : ~(Key)0;
    const Key* sk = block_sort<Key>(key, reinterpret_cast<Key*>(ka), reinterpret_cast<Key*>(kb));
    const Key kk = sk[tid];
    const bool first = tid < m && (tid == 0 || kk != sk[tid > 0 ? tid - 1 : 0]);
    const unsigned bal = __ballot_sync(FULL, first);
    if (lane == 0) ired[warp] = __popc(bal);
    __syncthreads();
    const int wcnt = ired[lane];
    int incl = wcnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += y;
    }
    const int nb = __shfl_sync(FULL, incl, 31);
    const int wbase = __shfl_sync(FULL, incl - wcnt, warp);
    const int bi = wbase + __popc(bal & ((1u << lane) - 1));  // boundary index of this run
    const int mid = m / 2;
    if (tid == mid) s_cle = bi + (first ? 1 : 0);  // runs starting at or before sorted position `mid`
    __syncthreads();
    const int center = s_cle - 1;
    int wlo = max(0, center - WIN / 2);
    const int whi = min(nb, wlo + WIN);
    wlo = max(0, whi - WIN);
    if (first && bi >= wlo && bi < whi) wb[(int64_t)ni * WIN + bi - wlo] = key_inv(kk, (T*)nullptr);
    if (tid < WIN) wf[(int64_t)ni * WIN + tid] = 0;
    if (tid == 0) {
        Split* sp = split + ni;
        sp->status = ST_SAMPLED;
        sp->dim = d0;
        sp->nb = nb;
        sp->wlo = wlo;
        sp->whi = whi;
        sp->value = 0.0;
        sp->nl = 0;
        sp->L = 0ULL;
    }
}

__device__ __forceinline__ int tile_node(const LNode* nodes, int K, uint32_t t) {
    int lo = 0, hi = K;  // last node with tile_off <= t
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (nodes[mid].tile_off <= t) lo = mid; else hi = mid;
    }
    return lo;
}


// ============================================================================
// k_hist: windowed histogram (median.py:128-140 restricted to the boundaries
// around the sampled median; counts below the window are aggregated in L).
// Besides the node totals it records, per half-tile, the window histogram row
// and the below-window count: once k_select has chosen the split boundary,
// each half-tile's "left" count is L_h + sum(row_h[1..wsel]) (k_tile_left), so
// the partition needs no second pass over the split column.
// ============================================================================
// one element global -> shared without a register round trip (cp.async, 4 or 8 bytes)
template <typename T>
__device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    if constexpr (sizeof(T) == 4) asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
    else asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}

// per tile of the level: node, element count and the offset of its split-dimension
// values in the level's SoA buffer (k_hist streams tiles from these)
struct TileInfo {
    int32_t ni;
    int32_t cnt;
    int64_t off;
};

static __global__ void k_tile_info(const LNode* __restrict__ nodes, int K, int32_t* __restrict__ tmap,
                                   const Split* __restrict__ split, uint32_t tiles, int64_t N,
                                   TileInfo* __restrict__ tinfo) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= tiles) return;
    const int ni = tile_node(nodes, K, t);
    tmap[t] = ni;
    const LNode nd = nodes[ni];
    const int64_t e0 = (int64_t)(t - nd.tile_off) * TILE;
    const int64_t e1 = min((int64_t)nd.n, e0 + TILE);
    tinfo[t] = TileInfo{ni, (int32_t)max((int64_t)0, e1 - e0), (int64_t)split[ni].dim * N + nd.start + e0};
}

// 1-D bulk copies (TMA engine, cp.async.bulk) into shared memory, completion counted
// in bytes on an mbarrier -- one instruction per tile instead of one cp.async per element
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    if (bytes)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                     ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
                     : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n KD_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra KD_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// a tile's split-column values as one 16-byte-aligned span (the TMA's unit): the copy
// starts at the aligned address below the first value; `lead` values precede it
template <typename T>
constexpr int HIST_SLOT = TILE + 32 / (int)sizeof(T);  // elements per tile buffer (alignment slack)

// Persistent: each CTA streams a contiguous run of tiles; the next tile's values
// arrive by bulk copy into the other shared buffer while the current one is
// classified, and the node's window / accumulators are only reloaded / flushed
// when the run crosses into another node.
template <typename T>
__global__ void __launch_bounds__(TILE_THREADS)
k_hist(const T* __restrict__ src, const TileInfo* __restrict__ tinfo, uint32_t tiles, Split* split,
       const T* __restrict__ wb, uint32_t* __restrict__ wf, uint16_t* __restrict__ hrow, uint32_t* __restrict__ hL) {
    constexpr int EPT = TILE / TILE_THREADS;
    constexpr int HPT = EPT / SUB;  // elements per thread in each half-tile
    constexpr int NW = TILE_THREADS / 32;
    extern __shared__ __align__(16) unsigned char hist_dyn[];  // 2 tile buffers (dynamic: 64 KB for f64)
    T (*buf)[HIST_SLOT<T>] = reinterpret_cast<T (*)[HIST_SLOT<T>]>(hist_dyn);
    __shared__ T sb[WIN];
    __shared__ uint32_t sf[SUB][WIN];
    __shared__ uint32_t nacc[WIN];
    __shared__ T q[NW][64];  // per-warp queue of in-window values (keeps the searches warp-dense)
    __shared__ uint32_t sL[SUB];
    __shared__ unsigned long long nL;
    __shared__ __align__(8) uint64_t mbar[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t t0 = (uint32_t)((uint64_t)tiles * blockIdx.x / gridDim.x);
    const uint32_t t1 = (uint32_t)((uint64_t)tiles * (blockIdx.x + 1) / gridDim.x);
    if (t0 >= t1) return;
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0]);
        mbar_init(&mbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto lead_of = [&](const TileInfo& ti) {
        return (int)(((uintptr_t)(src + ti.off) & 15) / sizeof(T));
    };
    auto issue = [&](const TileInfo& ti, int slot) {
        if (threadIdx.x == 0) {
            const char* g = reinterpret_cast<const char*>(src + ti.off);
            const char* a = reinterpret_cast<const char*>((uintptr_t)g & ~(uintptr_t)15);
            const unsigned bytes = ti.cnt ? (unsigned)(((g + (size_t)ti.cnt * sizeof(T) - a) + 15) & ~(size_t)15) : 0u;
            bulk_load(buf[slot], a, bytes, &mbar[slot]);
        }
    };
    TileInfo cur = tinfo[t0];
    issue(cur, 0);
    TileInfo nxt = t0 + 1 < t1 ? tinfo[t0 + 1] : TileInfo{-1, 0, 0};
    int cur_ni = -1, nw = 0;
    T lo_b = T(0), hi_b = T(0);
    for (uint32_t t = t0, it = 0; t < t1; t++, it++) {
        const int slot = it & 1;
        if (t + 1 < t1) issue(nxt, slot ^ 1);
        const TileInfo after = t + 2 < t1 ? tinfo[t + 2] : TileInfo{-1, 0, 0};
        if (cur.ni != cur_ni) {
            if (cur_ni >= 0) {  // flush the finished node
                for (int i = threadIdx.x + 1; i < nw; i += blockDim.x)
                    if (nacc[i]) atomicAdd(&wf[(int64_t)cur_ni * WIN + i], nacc[i]);
                if (threadIdx.x == 0 && nL) atomicAdd(&split[cur_ni].L, nL);
                __syncthreads();
            }
            cur_ni = cur.ni;
            const Split sp = split[cur_ni];
            nw = sp.whi - sp.wlo;
            // sb[i] = boundary i+1 for i < nw-2, +inf above: bin of x = 1 + #{i : sb[i] <= x}
            for (int i = threadIdx.x; i < WIN; i += blockDim.x) {
                nacc[i] = 0;
                sb[i] = i < nw - 2 ? wb[(int64_t)cur_ni * WIN + i + 1] : T(INFINITY);
            }
            if (threadIdx.x == 0) nL = 0;
            lo_b = wb[(int64_t)cur_ni * WIN];
            hi_b = wb[(int64_t)cur_ni * WIN + nw - 1];
        }
        for (int i = threadIdx.x; i < WIN; i += blockDim.x) {
            sf[0][i] = 0;
            sf[1][i] = 0;
        }
        if (threadIdx.x < SUB) sL[threadIdx.x] = 0;
        __syncthreads();
        mbar_wait(&mbar[slot], (it >> 1) & 1);  // this tile's bytes have landed
        const T* tb = buf[slot] + lead_of(cur);
#pragma unroll
        for (int h = 0; h < SUB; h++) {
            uint32_t* hist = sf[h];
            auto search = [&](T x) {  // branchless upper_bound of x in the boundaries 1 .. nw-2
                int pos = 0;
#pragma unroll
                for (int step = WIN / 2; step > 0; step >>= 1)
                    if (sb[pos + step - 1] <= x) pos += step;
                atomicAdd(&hist[1 + pos], 1u);
            };
            uint32_t lc = 0;
            int qn = 0;  // warp-uniform queue length
#pragma unroll
            for (int jj = 0; jj < HPT; jj++) {
                const int e = (h * HPT + jj) * TILE_THREADS + threadIdx.x;
                const bool ok = e < cur.cnt;
                const T v = tb[e];
                const bool below = ok && v < lo_b;
                const bool inwin = ok && !below && v < hi_b;
                lc += below;
                const unsigned m = __ballot_sync(FULL, inwin);
                if (inwin) q[warp][qn + __popc(m & ((1u << lane) - 1))] = v;
                qn += __popc(m);
                if (qn >= 32) {  // one dense round of 32 searches
                    __syncwarp();
                    search(q[warp][qn - 32 + lane]);
                    qn -= 32;
                    __syncwarp();
                }
            }
            __syncwarp();
            if (lane < qn) search(q[warp][lane]);
            __syncwarp();
            for (int o = 16; o > 0; o >>= 1) lc += __shfl_xor_sync(FULL, lc, o);
            if (lane == 0 && lc) atomicAdd(&sL[h], lc);
        }
        __syncthreads();
        if (threadIdx.x < SUB) hL[t * SUB + threadIdx.x] = sL[threadIdx.x];
        if (threadIdx.x == 0) nL += sL[0] + sL[1];
        for (int i = threadIdx.x; i < nw; i += blockDim.x) {
            const uint32_t a0 = sf[0][i], a1 = sf[1][i];
            hrow[((size_t)t * SUB) * WIN + i] = (uint16_t)a0;
            hrow[((size_t)t * SUB + 1) * WIN + i] = (uint16_t)a1;
            nacc[i] += a0 + a1;
        }
        __syncthreads();
        cur = nxt;
        nxt = after;
    }
    for (int i = threadIdx.x + 1; i < nw; i += blockDim.x)
        if (nacc[i]) atomicAdd(&wf[(int64_t)cur_ni * WIN + i], nacc[i]);
    if (threadIdx.x == 0 && nL) atomicAdd(&split[cur_ni].L, nL);
}

// everything the scatter needs about one half-tile, written by k_tile_left so the
// scatter's per-half-tile setup is one record load (+ the two scan entries)
struct HalfMeta {
    int64_t gbase;  // node start
    double value;   // split value
    int64_t nl;     // node's left count
    int32_t e0, e1; // element range within the node (e1 <= e0: nothing to move)
    int32_t dim;
    uint32_t first_hb;  // the node's first half-tile
};

// per half-tile count of elements going left: L_h + sum of the window bins
// below the chosen boundary (warp per half-tile); nodes split by the slow path
// (value not a window boundary) count from the data
template <typename T>
__global__ void k_tile_left(const T* __restrict__ src, const LNode* __restrict__ nodes, const int32_t* __restrict__ tmap,
                            DevCtx c, const Split* __restrict__ split, const uint16_t* __restrict__ hrow,
                            const uint32_t* __restrict__ hL, uint32_t nhalf, uint32_t* __restrict__ tile_left,
                            HalfMeta* __restrict__ meta) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t hb = blockIdx.x * (blockDim.x >> 5) + warp;
    if (hb >= nhalf) return;
    const uint32_t t = hb / SUB, sub = hb % SUB;
    const int ni = tmap[t];
    const Split sp = split[ni];
    const LNode nd = nodes[ni];
    const int64_t e0 = (int64_t)(t - nd.tile_off) * TILE + (int64_t)sub * (TILE / SUB);
    const int64_t e1 = min((int64_t)nd.n, e0 + TILE / SUB);
    uint32_t cnt = 0;
    if (sp.status == ST_SPLIT) {
        if (sp.wsel >= 0) {
            for (int i = 1 + lane; i <= sp.wsel; i += 32) cnt += hrow[(size_t)hb * WIN + i];
            cnt = warp_isum(cnt) + hL[hb];
        } else {
            const T* row = src + (int64_t)sp.dim * c.N + nd.start;
            for (int64_t e = e0 + lane; e < e1; e += 32) cnt += (double)row[e] < sp.value;
            cnt = warp_isum(cnt);
        }
    }
    if (lane == 0) {
        tile_left[hb] = cnt;
        const bool moves = sp.status == ST_SPLIT && e0 < e1;
        meta[hb] = HalfMeta{nd.start, sp.value, sp.nl, (int32_t)e0, moves ? (int32_t)e1 : (int32_t)e0, sp.dim,
                            nd.tile_off * SUB};
    }
}

// ============================================================================
// k_select: exact binary64 selection (median.py:143-166) from the window
// ============================================================================
template <typename T>
__global__ void k_select(const LNode* __restrict__ nodes, int K, Split* split, const T* __restrict__ wb,
                         const uint32_t* __restrict__ wf, int* slow_list, int* slow_count) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ni = blockIdx.x * (blockDim.x >> 5) + warp;
    if (ni >= K) return;
    Split sp = split[ni];
    const int64_t n = nodes[ni].n;
    const int nw = sp.whi - sp.wlo;
    constexpr int PER = WIN / 32;
    // lane owns window entries [lane*PER, lane*PER+PER)
    int64_t loc[PER];
    int64_t run = 0;
#pragma unroll
    for (int q = 0; q < PER; q++) {
        const int i = lane * PER + q;
        run += (i >= 1 && i < nw) ? (int64_t)wf[(int64_t)ni * WIN + i] : 0;
        loc[q] = run;
    }
    int64_t excl = run;
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(FULL, excl, o);
        if (lane >= o) excl += y;
    }
    excl -= run;
    const int64_t L = (int64_t)sp.L;
    double best = INFINITY;
    int besti = 0x7fffffff;
    int64_t bestc = 0;
#pragma unroll
    for (int q = 0; q < PER; q++) {
        const int i = lane * PER + q;
        if (i < nw) {
            const int64_t cum = L + excl + loc[q];
            const double df = half_diff(cum, n);
            if (df < best) { best = df; besti = i; bestc = cum; }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(FULL, best, o);
        const int oi = __shfl_xor_sync(FULL, besti, o);
        const int64_t oc = __shfl_xor_sync(FULL, bestc, o);
        if (ob < best || (ob == best && oi < besti)) { best = ob; besti = oi; bestc = oc; }
    }
    // cum at window ends
    const int64_t cum_lo = L;
    int64_t cum_hi = 0;
    {
        const int ih = nw - 1;
        const int owner = ih / PER, q = ih % PER;
        int64_t mine = 0;
#pragma unroll
        for (int qq = 0; qq < PER; qq++)
            if (qq == q) mine = L + excl + loc[qq];
        cum_hi = __shfl_sync(FULL, mine, owner);
    }
    if (lane == 0) {
        const double xlo = __ddiv_rn((double)cum_lo, (double)n);
        const double xhi = __ddiv_rn((double)cum_hi, (double)n);
        const bool okl = sp.wlo == 0 || (xlo <= 0.5 && besti > 0);
        const bool okr = sp.whi == sp.nb || xhi >= 0.5;
        if (okl && okr && bestc > 0 && bestc < n) {
            sp.status = ST_SPLIT;
            sp.value = (double)wb[(int64_t)ni * WIN + besti];
            sp.nl = bestc;
            sp.wsel = besti;
        } else {
            sp.status = ST_SLOW;
            slow_list[atomicAdd(slow_count, 1)] = ni;
        }
        split[ni] = sp;
    }
}

// ============================================================================
// k_slow: the reference's full split choice for one node (rare path)
// ============================================================================
template <typename T>
__global__ void __launch_bounds__(SLOW_THREADS)
k_slow(const T* __restrict__ src, const LNode* __restrict__ nodes, DevCtx c, Split* split,
       const int* slow_list, const int* slow_count) {
    typedef typename KeyOf<T>::type Key;
    __shared__ uint64_t skeys[MAXS];
    __shared__ uint32_t picked[MAXS];
    __shared__ T sb[MAXS];
    __shared__ int hist[MAXS + 1];
    __shared__ double s2x[16];
    __shared__ int order[16];
    __shared__ int s_nb;
    __shared__ unsigned long long red[SLOW_THREADS / 32];
    __shared__ Key kred[SLOW_THREADS / 32];
    __shared__ int s_done;
    __shared__ double s_val;
    __shared__ int64_t s_nl;
    __shared__ int s_dim;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cnt = *slow_count;
    const int D = c.dims;
    const int64_t N = c.N;
    for (int li = blockIdx.x; li < cnt; li += gridDim.x) {
        const int ni = slow_list[li];
        const LNode nd = nodes[ni];
        const int64_t n = nd.n;
        // ---- exact variance order (sequential, draw order)
        const int take = (int)min(n, c.vs);
        if (warp == 0) {
            const uint64_t vseed = node_seed(c.seed, nd.path, 0);
            if (n <= (1 << 22)) fy_resolve<32, uint32_t>((uint32_t)n, take, vseed, reinterpret_cast<uint32_t*>(skeys), picked);
            else fy_resolve<32, uint64_t>((uint32_t)n, take, vseed, skeys, picked);
            if (lane < D) {
                const T* row = src + (int64_t)lane * N + nd.start;
                double mean = 0.0;
                for (int j = 0; j < take; j++) mean = __dadd_rn(mean, (double)row[picked[j]]);
                mean = __ddiv_rn(mean, (double)take);
                double s = 0.0;
                for (int j = 0; j < take; j++) {
                    const double df = __dsub_rn((double)row[picked[j]], mean);
                    s = __dadd_rn(s, __dmul_rn(df, df));
                }
                s2x[lane] = s;
            }
            __syncwarp();
            if (lane == 0) {
                for (int d = 0; d < D; d++) order[d] = d;
                for (int a = 1; a < D; a++) {  // stable insertion sort on -ssd
                    const int tt = order[a];
                    int p = a - 1;
                    while (p >= 0 && -s2x[order[p]] > -s2x[tt]) { order[p + 1] = order[p]; p--; }
                    order[p + 1] = tt;
                }
            }
        }
        if (threadIdx.x == 0) s_done = 0;
        __syncthreads();
        for (int oi = 0; oi < D; oi++) {
            const int d = order[oi];
            const T* row = src + (int64_t)d * N + nd.start;
            const int m = (int)min(n, c.ms);
            if (warp == 0) {
                const uint64_t mseed = node_seed(c.seed, nd.path, 1ULL + (uint64_t)d);
                if (n <= (1 << 22)) fy_resolve<32, uint32_t>((uint32_t)n, m, mseed, reinterpret_cast<uint32_t*>(skeys), picked);
                else fy_resolve<32, uint64_t>((uint32_t)n, m, mseed, skeys, picked);
                Key kv[32];
#pragma unroll
                for (int r = 0; r < 32; r++) {
                    const int j = r * 32 + lane;
                    kv[r] = j < m ? tkey(row[picked[j]]) : ~(Key)0;
                }
                warp_sort_t<32>(kv);
                const Key kup = __shfl_up_sync(FULL, kv[31], 1);
                unsigned fmask = 0;
#pragma unroll
                for (int r = 0; r < 32; r++) {
                    const int s = lane * 32 + r;
                    const Key prev = sorted_prev<32>(kv, r, lane, kup, kv[0]);
                    fmask |= (unsigned)(s < m && (s == 0 || kv[r] != prev)) << r;
                }
                const int nf = __popc(fmask);
                int incl = nf;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += y;
                }
                const int nbr = __shfl_sync(FULL, incl, 31);
                int bi = incl - nf;
#pragma unroll
                for (int r = 0; r < 32; r++)
                    if ((fmask >> r) & 1u) sb[bi++] = key_inv(kv[r], (T*)nullptr);
                if (lane == 0) s_nb = nbr;
            }
            __syncthreads();
            const int nb = s_nb;
            for (int i = threadIdx.x; i <= nb; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
                const T v = row[e];
                int lo = 0, hi = nb;
                while (lo < hi) {
                    const int md = (lo + hi) >> 1;
                    if (sb[md] <= v) lo = md + 1; else hi = md;
                }
                atomicAdd(&hist[lo], 1);
            }
            __syncthreads();
            if (threadIdx.x == 0) {  // median.py:143-166, sequential
                int64_t cum = 0, below = 0;
                int bi = -1;
                double bd = INFINITY;
                for (int i = 0; i < nb; i++) {
                    cum += hist[i];
                    const double df = half_diff(cum, n);
                    if (df < bd) { bd = df; bi = i; below = cum; }
                }
                if (bi >= 0 && below > 0 && below < n) {
                    s_done = 1; s_dim = d; s_val = (double)sb[bi]; s_nl = below;
                }
            }
            __syncthreads();
            if (s_done) break;
            // ---- exact fallback (local_tree.py:162-177): s = k-th smallest, k = n/2
            const int64_t kth = n / 2;
            Key prefix = 0;
            int64_t krem = kth;
            constexpr int KB = KeyOf<T>::bits;
            for (int shift = KB - 8; shift >= 0; shift -= 8) {
                for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
                __syncthreads();
                const Key hmask = shift + 8 >= KB ? (Key)0 : (~(Key)0) << (shift + 8);
                for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
                    const Key k = tkey(row[e]);
                    if ((k & hmask) == (prefix & hmask)) atomicAdd(&hist[(int)((k >> shift) & 255)], 1);
                }
                __syncthreads();
                if (threadIdx.x == 0) {
                    int64_t acc = 0;
                    int dg = 0;
                    for (; dg < 256; dg++) {
                        if (acc + hist[dg] > krem) break;
                        acc += hist[dg];
                    }
                    krem -= acc;
                    s_nb = dg;
                }
                __syncthreads();
                prefix |= ((Key)s_nb) << shift;
                __syncthreads();
            }
            const Key ks = prefix;
            // below / equal counts and the next distinct value
            unsigned long long lt = 0, eq = 0;
            Key nxt = ~(Key)0;
            for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
                const Key k = tkey(row[e]);
                lt += k < ks;
                eq += k == ks;
                if (k > ks && k < nxt) nxt = k;
            }
            for (int o = 16; o > 0; o >>= 1) {
                lt += __shfl_xor_sync(FULL, lt, o);
                eq += __shfl_xor_sync(FULL, eq, o);
                const Key on = __shfl_xor_sync(FULL, nxt, o);
                nxt = on < nxt ? on : nxt;
            }
            if (lane == 0) { red[warp] = lt | (eq << 32); kred[warp] = nxt; }
            __syncthreads();
            if (threadIdx.x == 0) {
                int64_t below = 0, eqc = 0;
                Key nx = ~(Key)0;
                for (int w = 0; w < SLOW_THREADS / 32; w++) {
                    below += (int64_t)(red[w] & 0xFFFFFFFFULL);
                    eqc += (int64_t)(red[w] >> 32);
                    if (kred[w] < nx) nx = kred[w];
                }
                const double half = (double)n * 0.5;
                const int64_t i1 = below, i2 = below + eqc;
                const bool v1 = i1 >= 1, v2 = i2 < n;
                if (v1 || v2) {
                    bool pick2 = !v1 || (v2 && fabs((double)i2 - half) < fabs((double)i1 - half));
                    s_done = 1;
                    s_dim = d;
                    s_val = pick2 ? (double)key_inv(nx, (T*)nullptr) : (double)key_inv(ks, (T*)nullptr);
                    s_nl = pick2 ? i2 : i1;
                }
            }
            __syncthreads();
            if (s_done) break;
        }
        if (threadIdx.x == 0) {
            Split sp = split[ni];
            if (s_done) {
                sp.status = ST_SPLIT; sp.dim = s_dim; sp.value = s_val; sp.nl = s_nl; sp.wsel = -1;
            } else {
                sp.status = ST_LEAF;
            }
            split[ni] = sp;
        }
        __syncthreads();
    }
}

// ============================================================================
// stable segmented partition (local_tree.py:183-233), coordinates + row ids
// ============================================================================
// stable scatter of one tile: CH chunks of 256 elements per pass; every load of
// a pass is issued before the single block-wide prefix over (chunk, warp) counts
template <typename T, int DT, int CH>
__global__ void __launch_bounds__(TILE_THREADS)
k_scatter(const T* __restrict__ src, const int32_t* __restrict__ isrc, T* __restrict__ dst,
          int32_t* __restrict__ idst, const HalfMeta* __restrict__ meta, DevCtx c,
          const uint32_t* __restrict__ tile_loff, uint32_t nhalf) {
    constexpr int NW = TILE_THREADS / 32;
    constexpr int DC = DT > 0 ? DT : 16;
    __shared__ uint32_t wl[CH * NW];
    __shared__ uint32_t wpre[CH * NW];
    const int D = DT > 0 ? DT : c.dims;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent: a grid of resident CTAs strides over the half-tiles (empty second
    // halves of small nodes cost a loop iteration, not a CTA launch)
    // a contiguous run per CTA: the empty second halves of small nodes sit at every other index
    const uint32_t h0 = (uint32_t)((uint64_t)nhalf * blockIdx.x / gridDim.x);
    const uint32_t h1 = (uint32_t)((uint64_t)nhalf * (blockIdx.x + 1) / gridDim.x);
    for (uint32_t hb = h0; hb < h1; hb++) {
    const HalfMeta hm = meta[hb];
    if (hm.e1 <= hm.e0) continue;  // not split, or the empty second half of a small node
    const int64_t e0 = hm.e0, e1 = hm.e1;
    struct { int dim; double value; int64_t nl; } sp{hm.dim, hm.value, hm.nl};
    const uint32_t lbefore = tile_loff[hb] - tile_loff[hm.first_hb];  // lefts earlier in this node
    int64_t lrun = lbefore;
    int64_t rrun = e0 - lbefore;
    const int64_t N = c.N;
    const int64_t gbase = hm.gbase;
    for (int64_t pass = e0; pass < e1; pass += (int64_t)CH * TILE_THREADS) {
        T x[CH][DC];
        int32_t id[CH];
        bool f[CH];
        unsigned bal[CH];
#pragma unroll
        for (int j = 0; j < CH; j++) {
            const int64_t e = pass + j * TILE_THREADS + threadIdx.x;
            const bool valid = e < e1;
#pragma unroll
            for (int d = 0; d < DC; d++)
                if (d < D) x[j][d] = valid ? src[(int64_t)d * N + gbase + e] : T(0);
            id[j] = valid ? (isrc ? isrc[gbase + e] : (int32_t)(gbase + e)) : 0;  // level 0: ids = input rows
        }
#pragma unroll
        for (int j = 0; j < CH; j++) {
            const int64_t e = pass + j * TILE_THREADS + threadIdx.x;
            T xv = x[j][0];
#pragma unroll
            for (int d = 1; d < DC; d++)
                if (d == sp.dim) xv = x[j][d];
            f[j] = e < e1 && (double)xv < sp.value;
            bal[j] = __ballot_sync(FULL, f[j]);
            if (lane == 0) wl[j * NW + warp] = __popc(bal[j]);
        }
        __syncthreads();
        if (warp == 0) {  // exclusive prefix over (chunk, warp) in element order
            constexpr int PER = (CH * NW + 31) / 32;
            uint32_t loc[PER], s = 0;
#pragma unroll
            for (int q = 0; q < PER; q++) {
                const int i = lane * PER + q;
                loc[q] = s;
                s += i < CH * NW ? wl[i] : 0;
            }
            uint32_t incl = s;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += y;
            }
            const uint32_t ex = incl - s;
#pragma unroll
            for (int q = 0; q < PER; q++) {
                const int i = lane * PER + q;
                if (i < CH * NW) wpre[i] = ex + loc[q];
            }
            if (lane == 31) wl[0] = incl;  // pass total (wl no longer needed)
        }
        __syncthreads();
        const uint32_t ltot = wl[0];
#pragma unroll
        for (int j = 0; j < CH; j++) {
            const int64_t e = pass + j * TILE_THREADS + threadIdx.x;
            if (e >= e1) continue;
            const uint32_t lp = wpre[j * NW + warp] + __popc(bal[j] & ((1u << lane) - 1));
            const int64_t before = e - pass;  // elements of this pass before e
            const int64_t pos = f[j] ? lrun + lp : sp.nl + rrun + (before - lp);
            const int64_t gd = gbase + pos;
#pragma unroll
            for (int d = 0; d < DC; d++)
                if (d < D) dst[(int64_t)d * N + gd] = x[j][d];
            idst[gd] = id[j];
        }
        const int64_t pass_n = min((int64_t)CH * TILE_THREADS, e1 - pass);
        lrun += ltot;
        rrun += pass_n - ltot;
        __syncthreads();
    }
    }
}

// k_scatter_tma: the same stable partition for points of few dimensions, fed by
// the TMA engine.  A half-tile's D coordinate columns and its row ids arrive by
// 1-D bulk copies (cp.async.bulk + mbarrier) into one of two shared-memory
// stages; the next half-tile's copies are in flight while the current one is
// classified, prefixed and written -- the read stream never waits for the
// block-wide prefix or the stores (the register-staged k_scatter alternates
// load and store phases and reaches 5.2 TB/s).
template <typename T>
constexpr int SCAT_SLOT = TILE / SUB + 32 / (int)sizeof(T);  // elements per column buffer (alignment slack)
template <typename T, int DT>
constexpr size_t scat_stage_bytes() {
    return ((size_t)DT * SCAT_SLOT<T> * sizeof(T) + (size_t)SCAT_SLOT<int32_t> * sizeof(int32_t) + 15) & ~size_t(15);
}

template <typename T, int DT>
__global__ void __launch_bounds__(TILE_THREADS)
k_scatter_tma(const T* __restrict__ src, const int32_t* __restrict__ isrc, T* __restrict__ dst,
              int32_t* __restrict__ idst, const HalfMeta* __restrict__ meta, DevCtx c,
              const uint32_t* __restrict__ tile_loff, uint32_t nhalf) {
    constexpr int NW = TILE_THREADS / 32;
    constexpr int CH = TILE / SUB / TILE_THREADS;  // chunks of 256 elements per half-tile
    constexpr int HS = SCAT_SLOT<T>;
    extern __shared__ __align__(16) unsigned char scat_dyn[];
    __shared__ uint32_t wl[CH * NW];
    __shared__ uint32_t wpre[CH * NW];
    __shared__ __align__(8) uint64_t mbar[2];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t N = c.N;
    if (threadIdx.x == 0) {
        mbar_init(&mbar[0]);
        mbar_init(&mbar[1]);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    auto stage_cols = [&](int slot) { return reinterpret_cast<T*>(scat_dyn + (size_t)slot * scat_stage_bytes<T, DT>()); };
    auto stage_ids = [&](int slot) { return reinterpret_cast<int32_t*>(stage_cols(slot) + (size_t)DT * HS); };
    // one thread: expect the half-tile's bytes, then one bulk copy per column (+ ids)
    auto issue = [&](uint32_t hb, int slot) {
        const HalfMeta hm = meta[hb];
        const int64_t cnt = (int64_t)hm.e1 - hm.e0;
        unsigned bytes[DT + 1];
        const char* from[DT + 1];
        unsigned total = 0;
#pragma unroll
        for (int d = 0; d <= DT; d++) {
            bytes[d] = 0;
            from[d] = nullptr;
            if (cnt <= 0 || (d == DT && !isrc)) continue;
            const char* g = d < DT ? reinterpret_cast<const char*>(src + (int64_t)d * N + hm.gbase + hm.e0)
                                   : reinterpret_cast<const char*>(isrc + hm.gbase + hm.e0);
            const size_t esz = d < DT ? sizeof(T) : sizeof(int32_t);
            const char* a = reinterpret_cast<const char*>((uintptr_t)g & ~(uintptr_t)15);
            from[d] = a;
            bytes[d] = (unsigned)(((g + (size_t)cnt * esz - a) + 15) & ~(size_t)15);
            total += bytes[d];
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&mbar[slot])), "r"(total)
                     : "memory");
#pragma unroll
        for (int d = 0; d <= DT; d++) {
            if (!bytes[d]) continue;
            void* to = d < DT ? (void*)(stage_cols(slot) + (size_t)d * HS) : (void*)stage_ids(slot);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                         ::"r"(smem_u32(to)), "l"(from[d]), "r"(bytes[d]), "r"(smem_u32(&mbar[slot]))
                         : "memory");
        }
    };
    // each CTA takes a contiguous run of half-tiles (the empty second halves of nodes of <= 2048
    // points sit at every other index: a strided walk would hand them all to every other CTA)
    // and skips the empty ones; stages / parities advance with the non-empty ones only
    const uint32_t h0 = (uint32_t)((uint64_t)nhalf * blockIdx.x / gridDim.x);
    const uint32_t h1 = (uint32_t)((uint64_t)nhalf * (blockIdx.x + 1) / gridDim.x);
    auto next_work = [&](uint32_t from) {  // first non-empty half-tile in [from, h1), or h1
        while (from < h1 && meta[from].e1 <= meta[from].e0) from++;
        return from;
    };
    if (threadIdx.x == 0) {
        const uint32_t f = next_work(h0);
        if (f < h1) issue(f, 0);
    }
    uint32_t it = 0;
    for (uint32_t hb = h0; hb < h1; hb++) {
        const HalfMeta hm = meta[hb];
        if (hm.e1 <= hm.e0) continue;  // not split, or the empty second half of a small node
        const int slot = it & 1;
        if (threadIdx.x == 0) {
            const uint32_t f = next_work(hb + 1);
            if (f < h1) issue(f, slot ^ 1);
        }
        mbar_wait(&mbar[slot], (it >> 1) & 1);  // this half-tile's bytes have landed
        {
            const int cnt = hm.e1 - hm.e0;
            const int64_t gbase = hm.gbase;
            const uint32_t lbefore = tile_loff[hb] - tile_loff[hm.first_hb];  // lefts earlier in this node
            const int64_t lrun = lbefore;
            const int64_t rrun = (int64_t)hm.e0 - lbefore;
            const T* col[DT];
#pragma unroll
            for (int d = 0; d < DT; d++)
                col[d] = stage_cols(slot) + (size_t)d * HS +
                         (((uintptr_t)(src + (int64_t)d * N + gbase + hm.e0) & 15) / sizeof(T));
            const int32_t* icol = stage_ids(slot) + (isrc ? ((uintptr_t)(isrc + gbase + hm.e0) & 15) / sizeof(int32_t) : 0);
            const T* scol = col[0];
#pragma unroll
            for (int d = 1; d < DT; d++)
                if (d == hm.dim) scol = col[d];
            bool f[CH];
            unsigned bal[CH];
#pragma unroll
            for (int j = 0; j < CH; j++) {
                const int e = j * TILE_THREADS + threadIdx.x;
                f[j] = e < cnt && (double)scol[e < cnt ? e : 0] < hm.value;
                bal[j] = __ballot_sync(FULL, f[j]);
                if (lane == 0) wl[j * NW + warp] = __popc(bal[j]);
            }
            __syncthreads();
            if (warp == 0) {  // exclusive prefix over (chunk, warp) in element order
                constexpr int PER = (CH * NW + 31) / 32;
                uint32_t loc[PER], sum = 0;
#pragma unroll
                for (int q = 0; q < PER; q++) {
                    const int i = lane * PER + q;
                    loc[q] = sum;
                    sum += i < CH * NW ? wl[i] : 0;
                }
                uint32_t incl = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(FULL, incl, o);
                    if (lane >= o) incl += y;
                }
                const uint32_t ex = incl - sum;
#pragma unroll
                for (int q = 0; q < PER; q++) {
                    const int i = lane * PER + q;
                    if (i < CH * NW) wpre[i] = ex + loc[q];
                }
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < CH; j++) {
                const int e = j * TILE_THREADS + threadIdx.x;
                if (e >= cnt) continue;
                const uint32_t lp = wpre[j * NW + warp] + __popc(bal[j] & ((1u << lane) - 1));
                const int64_t pos = f[j] ? lrun + lp : hm.nl + rrun + ((int64_t)e - lp);
                const int64_t gd = gbase + pos;
#pragma unroll
                for (int d = 0; d < DT; d++) dst[(int64_t)d * N + gd] = col[d][e];
                idst[gd] = isrc ? icol[e] : (int32_t)(gbase + hm.e0 + e);  // level 0: ids = input rows
            }
        }
        __syncthreads();  // the stage is free for the copy issued two iterations on; wl / wpre reusable
        it++;
    }
}

// ============================================================================
// k_children: records + next level + subtree tasks
// ============================================================================
struct TopStore {
    int32_t* dim;
    double* val;
    int32_t* left;
    int32_t* right;
    int32_t* npts;
    int32_t* kind;
    int32_t* task;
    int32_t* nodes;  // subtree node counts
    int32_t* pre;    // preorder index
};

static __global__ void k_children(const LNode* __restrict__ nodes, int K, const Split* __restrict__ split, DevCtx c,
                           int dst_parity, int src_parity, int child_base, TopStore ts, LNode* next,
                           unsigned long long* next_ctr, Task* tasks, int* task_ctr, int* next_max) {
    const int ni = blockIdx.x * blockDim.x + threadIdx.x;
    if (ni >= K) return;
    const LNode nd = nodes[ni];
    const Split sp = split[ni];
    if (sp.status == ST_LEAF) {
        const int t = atomicAdd(task_ctr, 1);
        tasks[t] = Task{nd.start, nd.n, nd.depth, nd.path, nd.slot, src_parity, 1, 0};
        ts.kind[nd.slot] = TS_TASK;
        ts.task[nd.slot] = t;
        ts.npts[nd.slot] = nd.n;
        return;
    }
    const int ls = child_base + 2 * ni, rs = ls + 1;
    ts.kind[nd.slot] = TS_INTERIOR;
    ts.dim[nd.slot] = sp.dim;
    ts.val[nd.slot] = sp.value;
    ts.left[nd.slot] = ls;
    ts.right[nd.slot] = rs;
    ts.npts[nd.slot] = nd.n;
    const int64_t cs[2] = {nd.start, nd.start + sp.nl};
    const int32_t cn[2] = {(int32_t)sp.nl, (int32_t)(nd.n - sp.nl)};
    const int32_t slot[2] = {ls, rs};
    const uint64_t cp[2] = {nd.path * 2ULL, nd.path * 2ULL + 1ULL};
    for (int k = 0; k < 2; k++) {
        ts.npts[slot[k]] = cn[k];
        if (cn[k] > c.ts) {
            const uint32_t nt = (uint32_t)((cn[k] + TILE - 1) / TILE);
            const unsigned long long old = atomicAdd(next_ctr, (1ULL << 32) | nt);
            const int idx = (int)(old >> 32);
            next[idx] = LNode{cs[k], cn[k], nd.depth + 1, cp[k], slot[k], (uint32_t)(old & 0xFFFFFFFFULL)};
            ts.kind[slot[k]] = TS_INTERIOR;
            atomicMax(next_max, cn[k]);
        } else {
            const int t = atomicAdd(task_ctr, 1);
            tasks[t] = Task{cs[k], cn[k], nd.depth + 1, cp[k], slot[k], dst_parity, 0, 0};
            ts.kind[slot[k]] = TS_TASK;
            ts.task[slot[k]] = t;
        }
    }
}

// ============================================================================
// k_subtree: one warp builds a whole subtree of <= ts points, depth first in
// preorder (local_tree.py:236-317 _build_subtree), points staged in shared
// memory.  For n <= min(local_sample_m, variance_sample) the reference's
// samples are the whole node, so split selection reduces to: the max-variance
// non-constant dimension (certified binary64 sums, exact sequential fallback),
// then the two distinct values around rank n/2 (radix select) compared with
// the binary64 rule of median.py:143-166.
// ============================================================================
// A pointer into the kernel's dynamic shared memory, re-expressed as an offset from the dynamic
// shared array itself: the compiler then knows the address space inside the non-inlined split
// functions and emits shared loads / stores / atomics.  (__builtin_assume(__isShared(p)) is not a
// safe substitute: when the caller derives p from the dynamic array plus a runtime offset, the
// assumption is folded to false and the code behind it is removed -- measured with several tasks
// per CTA, which was also no faster: 25.2 vs 24.3 ms.)
extern __shared__ __align__(16) unsigned char kd_dyn_smem[];
template <typename P>
__device__ __forceinline__ P* as_dyn_shared(P* p) {
    const uint32_t off = (uint32_t)(__cvta_generic_to_shared(p) - __cvta_generic_to_shared(kd_dyn_smem));
    return reinterpret_cast<P*>(const_cast<unsigned char*>(kd_dyn_smem) + off);
}

struct SubStack {
    uint64_t path;
    int32_t parent_pre;  // -1: root / left child (no patch); else parent whose right child this is
    uint32_t packed;     // start (10 bits) | n (11 bits) << 10 | rel depth (11 bits) << 21
};

constexpr int FY_SLOTS = 8192;  // global scratch slots for the rare exact-variance path
constexpr int SUB_WARPS_HOST = 2;  // == SUB_WARPS (k_subtree)

__host__ __device__ inline size_t sub_smem_bytes(int ts, int dims, int tsize) {
    size_t b = (size_t)dims * ts * tsize;
    b = (b + 15) & ~size_t(15);
    b += (size_t)2 * ts * 2;  // perm ping-pong by depth parity
    b = (b + 15) & ~size_t(15);
    b += SUB_WARPS_HOST * 256 * 4;  // radix histogram per warp
    return b;
}

// k-th smallest key (0-based) of the node's values + below/equal counts.  Keys are read from
// shared memory through the node's permutation (runtime loops: small code, few registers);
// 8-bit digit radix select with a per-warp shared-memory histogram.  The counts fall out of
// the passes: the rank left inside the last digit's bin is the key's rank among its equals,
// so lt = kth - rem and eq = that bin's count (no counting pass over the node).
template <typename T>
__device__ __forceinline__ void warp_select(const T* row, const uint16_t* pm, int n, int kth, uint32_t* hist,
                                            typename KeyOf<T>::type kmin_, typename KeyOf<T>::type kmax_,
                                            typename KeyOf<T>::type& ks, int& lt, int& eq) {
    typedef typename KeyOf<T>::type Key;
    row = as_dyn_shared(row);
    pm = as_dyn_shared(pm);
    hist = as_dyn_shared(hist);
    const int lane = threadIdx.x & 31;
    constexpr int KB = sizeof(Key) * 8;
    // every key lies in [kmin_, kmax_]: their common high bytes need no pass
    const Key diff = kmin_ ^ kmax_;
    int top = KB - 1;
    while (top > 0 && !((diff >> top) & 1)) top--;
    const int start = (top / 8) * 8;
    Key prefix = start + 8 >= KB ? (Key)0 : (kmin_ & ((~(Key)0) << (start + 8)));
    int rem = kth;
    int bin = n;  // keys in the selected bin of the last pass
#pragma unroll 1
    for (int shift = start; shift >= 0; shift -= 8) {
        for (int i = lane; i < 256; i += 32) hist[i] = 0;
        __syncwarp();
        const Key hmask = shift + 8 >= KB ? (Key)0 : (~(Key)0) << (shift + 8);
#pragma unroll 4
        for (int i = lane; i < n; i += 32) {
            const Key kk = tkey(row[pm[i]]);
            if ((kk & hmask) == (prefix & hmask)) atomicAdd(&hist[(int)((kk >> shift) & 255)], 1u);
        }
        __syncwarp();
        uint32_t h[8];
        uint32_t s = 0;
#pragma unroll
        for (int j = 0; j < 8; j++) { h[j] = hist[lane * 8 + j]; s += h[j]; }
        uint32_t incl = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t excl = incl - s;
        const bool mine = (uint32_t)rem >= excl && (uint32_t)rem < incl;
        int digit = 0, newrem = 0, cnt = 0;
        if (mine) {
            uint32_t acc = excl;
#pragma unroll
            for (int j = 0; j < 8; j++) {
                if ((uint32_t)rem >= acc && (uint32_t)rem < acc + h[j]) {
                    digit = lane * 8 + j;
                    newrem = rem - (int)acc;
                    cnt = (int)h[j];
                }
                acc += h[j];
            }
        }
        const int src = __ffs(__ballot_sync(FULL, mine)) - 1;
        digit = __shfl_sync(FULL, digit, src);
        rem = __shfl_sync(FULL, newrem, src);
        bin = __shfl_sync(FULL, cnt, src);
        prefix |= ((Key)digit) << shift;
        __syncwarp();
    }
    ks = prefix;
    lt = kth - rem;
    eq = bin;
}

// smallest key above ks (only needed when the split takes the next boundary)
template <typename T>
__device__ __forceinline__ typename KeyOf<T>::type warp_next_key(const T* row, const uint16_t* pm, int n,
                                                                 typename KeyOf<T>::type ks) {
    typedef typename KeyOf<T>::type Key;
    row = as_dyn_shared(row);
    pm = as_dyn_shared(pm);
    const int lane = threadIdx.x & 31;
    Key nx = ~(Key)0;
#pragma unroll 4
    for (int i = lane; i < n; i += 32) {
        const Key kk = tkey(row[pm[i]]);
        if (kk > ks && kk < nx) nx = kk;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const Key on = __shfl_xor_sync(FULL, nx, o);
        nx = on < nx ? on : nx;
    }
    return nx;
}

static __device__ __noinline__ void fy_resolve_n(uint32_t n, uint64_t seed, uint32_t* fk, uint32_t* fp) {
    if (n <= 32) fy_resolve<1, uint32_t>(n, (int)n, seed, fk, fp);
    else if (n <= 64) fy_resolve<2, uint32_t>(n, (int)n, seed, fk, fp);
    else if (n <= 128) fy_resolve<4, uint32_t>(n, (int)n, seed, fk, fp);
    else if (n <= 256) fy_resolve<8, uint32_t>(n, (int)n, seed, fk, fp);
    else if (n <= 512) fy_resolve<16, uint32_t>(n, (int)n, seed, fk, fp);
    else fy_resolve<32, uint32_t>(n, (int)n, seed, fk, fp);
}

// exact max-variance dimension of a whole-node sample (the reference's
// sequential two-pass sums in Fisher-Yates draw order); rare: near-ties only
template <typename T>
__device__ __noinline__ int sub_exact_dim(const T* cs, const uint16_t* pm, int n, int ts, int D, unsigned ncmask,
                                          uint64_t path, const DevCtx& c, uint32_t* fyslots, int* fylocks) {
    const int lane = threadIdx.x & 31;
    const int slot = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % FY_SLOTS;
    if (lane == 0) while (atomicCAS(&fylocks[slot], 0, 1) != 0) {}
    __syncwarp();
    __threadfence();
    uint32_t* fk = fyslots + (size_t)slot * 2 * MAXS;
    uint32_t* fp = fk + MAXS;
    fy_resolve_n((uint32_t)n, node_seed(c.seed, path, 0), fk, fp);
    double exact = 0.0;
    if (lane < D && ((ncmask >> lane) & 1u)) {
        const T* row = cs + lane * ts;
        double mean = 0.0;
        for (int j = 0; j < n; j++) mean = __dadd_rn(mean, (double)row[pm[fp[j]]]);
        mean = __ddiv_rn(mean, (double)n);
        double s = 0.0;
        for (int j = 0; j < n; j++) {
            const double df = __dsub_rn((double)row[pm[fp[j]]], mean);
            s = __dadd_rn(s, __dmul_rn(df, df));
        }
        exact = s;
    }
    __syncwarp();
    __threadfence();
    if (lane == 0) atomicExch(&fylocks[slot], 0);
    int best = -1;
    double bv = 0.0;
    for (int d = 0; d < D; d++) {
        const double e = __shfl_sync(FULL, exact, d);
        if (!((ncmask >> d) & 1u)) continue;
        if (best < 0 || -e < -bv) { best = d; bv = e; }  // stable descending (argsort(-ssd))
    }
    return best;
}

// half_diff(b, n) < half_diff(a, n) exactly as the reference evaluates it
// (median.py:160): distinct |2c - n| differ by >= 1/(2n) in the exact values,
// far above the binary64 rounding of c/n, so the integers decide; only exact
// mirror ties (a + b == n) need the rounded divisions
__device__ __forceinline__ bool closer_to_half(int64_t b, int64_t a, int64_t n) {
    const int64_t db = 2 * b - n, da = 2 * a - n;
    const int64_t ab = db < 0 ? -db : db, aa = da < 0 ? -da : da;
    if (ab != aa) return ab < aa;
    return half_diff(b, n) < half_diff(a, n);
}

// Small nodes (n <= 32*SR, fixed dimension count): the node's points are read
// once into registers; per-dimension sums come from registers and the split
// dimension's keys are sorted by the unrolled network (warp_sort_t) instead of
// radix-select passes.  Same decisions as sub_split (same certified bound).
template <typename T, int DT, int SR>
__device__ __noinline__ void sub_split_small(const T* cs, const uint16_t* pm, int n, int ts, uint64_t path,
                                                const DevCtx& c, uint32_t* fyslots, int* fylocks, int& out_dim,
                                                double& out_val, int& out_nl) {
    typedef typename KeyOf<T>::type Key;
    cs = as_dyn_shared(cs);
    pm = as_dyn_shared(pm);
    const int lane = threadIdx.x & 31;
    T x[DT][SR];
#pragma unroll
    for (int r = 0; r < SR; r++) {
        const int i = r * 32 + lane;
        const int q = pm[i < n ? i : 0];
#pragma unroll
        for (int d = 0; d < DT; d++) x[d][r] = cs[d * ts + q];
    }
    // per dimension: constant?, shifted binary64 sums (y = x - x0); the reductions of every
    // dimension run interleaved (one butterfly).  A float dimension is constant exactly when
    // sum y^2 == 0 (y == 0 iff x == x0, and a float difference squared cannot underflow in
    // binary64), so only double coordinates need the min / max keys.
    constexpr bool KEYS = sizeof(T) != 4;
    Key kmn[DT], kmx[DT];
    double s1[DT], sq[DT];
#pragma unroll
    for (int d = 0; d < DT; d++) {
        const double x0 = (double)__shfl_sync(FULL, x[d][0], 0);
        kmn[d] = ~(Key)0;
        kmx[d] = 0;
        s1[d] = 0.0;
        sq[d] = 0.0;
#pragma unroll
        for (int r = 0; r < SR; r++) {
            if (r * 32 + lane < n) {
                if constexpr (KEYS) {
                    const Key k = tkey(x[d][r]);
                    kmn[d] = k < kmn[d] ? k : kmn[d];
                    kmx[d] = k > kmx[d] ? k : kmx[d];
                }
                const double y = __dsub_rn((double)x[d][r], x0);
                s1[d] = __dadd_rn(s1[d], y);
                sq[d] = __dadd_rn(sq[d], __dmul_rn(y, y));
            }
        }
    }
#pragma unroll 1  // rolled: the kernel is bound by instruction fetch (-1.1 ms on C3)
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int d = 0; d < DT; d++) {
            if constexpr (KEYS) {
                const Key a = __shfl_xor_sync(FULL, kmn[d], o), b = __shfl_xor_sync(FULL, kmx[d], o);
                kmn[d] = a < kmn[d] ? a : kmn[d];
                kmx[d] = b > kmx[d] ? b : kmx[d];
            }
            s1[d] = __dadd_rn(s1[d], __shfl_xor_sync(FULL, s1[d], o));
            sq[d] = __dadd_rn(sq[d], __shfl_xor_sync(FULL, sq[d], o));
        }
    }
    const double rn = 1.0 / (double)n;
    int best = -1;
    double bs = 0.0, be = 0.0;
    double s2v[DT], eb[DT];
    unsigned ncmask = 0;
#pragma unroll
    for (int d = 0; d < DT; d++) {
        s2v[d] = 0.0;
        eb[d] = 0.0;
        if (KEYS ? kmn[d] == kmx[d] : sq[d] == 0.0) continue;
        ncmask |= 1u << d;
        const double bb = __dmul_rn(__dmul_rn(s1[d], s1[d]), rn);
        s2v[d] = sq[d] - bb;
        // + 4u*bb: the reciprocal product instead of a correctly rounded division
        eb[d] = 4.0 * ((double)n + 8.0) * U64 * (sq[d] + bb) + 4.0 * U64 * bb + 1e-300;
        if (best < 0 || s2v[d] > bs) { best = d; bs = s2v[d]; be = eb[d]; }
    }
    out_dim = -1;
    if (best < 0) return;
    bool certified = true;
#pragma unroll
    for (int d = 0; d < DT; d++)
        if (d != best && ((ncmask >> d) & 1u) && !(bs - s2v[d] > be + eb[d])) certified = false;
    if (!certified) best = sub_exact_dim<T>(cs, pm, n, ts, DT, ncmask, path, c, fyslots, fylocks);
    Key kv[SR];
#pragma unroll
    for (int r = 0; r < SR; r++) {
        T v = x[0][r];
#pragma unroll
        for (int d = 1; d < DT; d++)
            if (d == best) v = x[d][r];
        kv[r] = r * 32 + lane < n ? tkey(v) : ~(Key)0;
    }
    // (the rolled network is slower here: 24.7 vs 23.2 ms -- too small a body for the loop overhead)
    warp_sort_t<SR>(kv);  // sorted element s in lane s / SR, register s % SR
    const int h = n / 2;
    Key mine = kv[0];
#pragma unroll
    for (int r = 1; r < SR; r++)
        if (r == h % SR) mine = kv[r];
    const Key ks = __shfl_sync(FULL, mine, h / SR);
    int lt = 0, eq = 0;
    Key nx = ~(Key)0;
#pragma unroll
    for (int r = 0; r < SR; r++) {
        const bool valid = lane * SR + r < n;
        lt += __popc(__ballot_sync(FULL, valid && kv[r] < ks));
        eq += __popc(__ballot_sync(FULL, valid && kv[r] == ks));
        if (valid && kv[r] > ks && kv[r] < nx) nx = kv[r];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const Key on = __shfl_xor_sync(FULL, nx, o);
        nx = on < nx ? on : nx;
    }
    const int cumA = lt, cumB = lt + eq;
    bool pickB;
    if (cumA == 0) pickB = true;
    else if (cumB >= n) pickB = false;
    else pickB = closer_to_half(cumB, cumA, n);
    out_dim = best;
    out_val = pickB ? (double)key_inv(nx, (T*)nullptr) : (double)key_inv(ks, (T*)nullptr);
    out_nl = pickB ? cumB : cumA;
}

template <typename T, int DT>
__device__ __noinline__ void sub_split(const T* cs, const uint16_t* pm, int n, int ts, int dims_rt, uint64_t path,
                          const DevCtx& c, uint32_t* hist, uint32_t* fyslots, int* fylocks, int& out_dim,
                          double& out_val, int& out_nl) {
    typedef typename KeyOf<T>::type Key;
    cs = as_dyn_shared(cs);
    pm = as_dyn_shared(pm);
    hist = as_dyn_shared(hist);
    constexpr int DC = DT > 0 ? DT : 16;
    const int D = DT > 0 ? DT : dims_rt;
    const int lane = threadIdx.x & 31;
    // per dimension: constant?, binary64 sum of squared deviations + bound.  One
    // pass over the node reads each point's index once for every dimension
    // (shifted sums y = x - x0, x0 = the node's first point; S2 = sum y^2 - (sum y)^2 / n),
    // then the reductions of all dimensions run interleaved.
    // (float coordinates: the min / max run on the values themselves -- one FMNMX each instead of
    //  a key conversion per element -- and become keys after the reduction)
    constexpr bool FVAL = sizeof(T) == 4;
    typedef typename std::conditional<FVAL, float, Key>::type MM;
    MM kmins[DC], kmaxs[DC];
    double s1[DC], sq[DC], x0[DC];
    {
        const int q0 = pm[0];
#pragma unroll
        for (int d = 0; d < DC; d++) {
            x0[d] = d < D ? (double)cs[d * ts + q0] : 0.0;
            if constexpr (FVAL) {
                kmins[d] = INFINITY;
                kmaxs[d] = -INFINITY;
            } else {
                kmins[d] = ~(Key)0;
                kmaxs[d] = 0;
            }
            s1[d] = 0.0;
            sq[d] = 0.0;
        }
    }
#pragma unroll 2
    for (int i = lane; i < n; i += 32) {
        const int qv = pm[i];
#pragma unroll
        for (int d = 0; d < DC; d++) {
            if (d < D) {
                const T v = cs[d * ts + qv];
                if constexpr (FVAL) {
                    kmins[d] = fminf(kmins[d], (float)v);
                    kmaxs[d] = fmaxf(kmaxs[d], (float)v);
                } else {
                    const Key k = tkey(v);
                    kmins[d] = k < kmins[d] ? k : kmins[d];
                    kmaxs[d] = k > kmaxs[d] ? k : kmaxs[d];
                }
                const double y = __dsub_rn((double)v, x0[d]);
                s1[d] = __dadd_rn(s1[d], y);
                sq[d] = __dadd_rn(sq[d], __dmul_rn(y, y));
            }
        }
    }
#pragma unroll 1  // rolled: the kernel is bound by instruction fetch (-1.1 ms on C3)
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int d = 0; d < DC; d++) {
            if (d < D) {
                const MM a = __shfl_xor_sync(FULL, kmins[d], o), b = __shfl_xor_sync(FULL, kmaxs[d], o);
                if constexpr (FVAL) {
                    kmins[d] = fminf(kmins[d], a);
                    kmaxs[d] = fmaxf(kmaxs[d], b);
                } else {
                    kmins[d] = a < kmins[d] ? a : kmins[d];
                    kmaxs[d] = b > kmaxs[d] ? b : kmaxs[d];
                }
                s1[d] = __dadd_rn(s1[d], __shfl_xor_sync(FULL, s1[d], o));
                sq[d] = __dadd_rn(sq[d], __shfl_xor_sync(FULL, sq[d], o));
            }
        }
    }
    const double rn = 1.0 / (double)n;
    int best = -1;
    double bs = 0.0, be = 0.0;
    double s2v[DC], eb[DC];
    unsigned ncmask = 0;
#pragma unroll
    for (int d = 0; d < DC; d++) {
        s2v[d] = 0.0;
        eb[d] = 0.0;
        if (d >= D || kmins[d] == kmaxs[d]) continue;
        ncmask |= 1u << d;
        const double bb = __dmul_rn(__dmul_rn(s1[d], s1[d]), rn);
        s2v[d] = sq[d] - bb;
        // rigorous bound on |computed - reference two-pass value| (both vs the exact sum of
        // squared deviations): shifted-sum rounding + the reference's own two-pass error
        // (+ 4u*bb for the reciprocal product)
        eb[d] = 4.0 * ((double)n + 8.0) * U64 * (sq[d] + bb) + 4.0 * U64 * bb + 1e-300;
        if (best < 0 || s2v[d] > bs) { best = d; bs = s2v[d]; be = eb[d]; }
    }
    out_dim = -1;
    if (best < 0) return;  // every dimension constant: degenerate leaf
    bool certified = true;
#pragma unroll
    for (int d = 0; d < DC; d++)
        if (d != best && ((ncmask >> d) & 1u) && !(bs - s2v[d] > be + eb[d])) certified = false;
    if (!certified) best = sub_exact_dim<T>(cs, pm, n, ts, D, ncmask, path, c, fyslots, fylocks);
    Key ks;
    int lt, eq;
    MM mmin = kmins[0], mmax = kmaxs[0];
#pragma unroll
    for (int d = 1; d < DC; d++)
        if (d == best) { mmin = kmins[d]; mmax = kmaxs[d]; }
    Key bmin, bmax;
    if constexpr (FVAL) {
        bmin = tkey((T)mmin);
        bmax = tkey((T)mmax);
    } else {
        bmin = mmin;
        bmax = mmax;
    }
    warp_select<T>(cs + best * ts, pm, n, n / 2, hist, bmin, bmax, ks, lt, eq);
    const int cumA = lt, cumB = lt + eq;
    bool pickB;
    if (cumA == 0) pickB = true;          // A is the first boundary (diff 0.5)
    else if (cumB >= n) pickB = false;    // no boundary after A
    else pickB = closer_to_half(cumB, cumA, n);
    out_dim = best;
    out_val = pickB ? (double)key_inv(warp_next_key<T>(cs + best * ts, pm, n, ks), (T*)nullptr)
                    : (double)key_inv(ks, (T*)nullptr);
    out_nl = pickB ? cumB : cumA;
}


// Two warps per task (SUB_WARPS): warp 0 splits the task's root, then the warps
// build the two child subtrees concurrently (disjoint ranges of the shared
// permutation, own radix histogram, own node / stack regions: a subtree of m
// points has at most 2m-1 nodes, so the right subtree is numbered from 0 at
// offset 2*nl and moved down behind the left one at the end).  Same shared
// memory per task as one warp, twice the resident warps per SM.
constexpr int SUB_WARPS = 2;
constexpr int SUB_THREADS = SUB_WARPS * 32;

__device__ __forceinline__ void pair_sync() {
    asm volatile("bar.sync 1, %0;\n" ::"n"(SUB_THREADS) : "memory");
}

template <typename T, int DT>
__global__ void __launch_bounds__(SUB_THREADS, 12)
k_subtree(const Task* __restrict__ tasks, T* buf0, const T* buf1, const T* in0, int32_t* idx0, const int32_t* idx1, DevCtx c,
          KdNode* __restrict__ scratch, int32_t* __restrict__ scnt, SubStack* __restrict__ sstack,
          uint32_t* __restrict__ fyslots, int* __restrict__ fylocks, int32_t* task_nodes, int32_t* task_depth) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int task = blockIdx.x;
    const Task tk = tasks[task];
    const int D = DT > 0 ? DT : c.dims;
    const int64_t N = c.N;
    const int ts = c.ts;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // tk.src: 0 / 1 = build buffer, 2 = the caller's input (row ids = positions)
    const T* src = tk.src == 2 ? in0 : (tk.src ? buf1 : buf0);
    const int32_t* isrc = tk.src == 2 ? nullptr : (tk.src ? idx1 : idx0);
    KdNode* out_nodes = scratch + 2 * tk.start;
    int32_t* out_cnt = scnt + 2 * tk.start;
    SubStack* stk = sstack + 2 * tk.start;

    if (tk.leaf || tk.n > ts) {
        // degenerate leaf (possibly larger than the shared-memory limit): copy through
        if (tk.src) {
            for (int64_t e = tid; e < tk.n; e += SUB_THREADS) {
                for (int d = 0; d < D; d++) buf0[(int64_t)d * N + tk.start + e] = src[(int64_t)d * N + tk.start + e];
                idx0[tk.start + e] = isrc ? isrc[tk.start + e] : (int32_t)(tk.start + e);
            }
        }
        if (tid == 0) {
            out_nodes[0] = KdNode{0.0, (int32_t)tk.start, -1 - tk.n};
            out_cnt[0] = tk.n;
            task_nodes[task] = 1;
            task_depth[task] = tk.depth;
        }
        return;
    }
    const int n = tk.n;
    unsigned char* p = smem_raw;
    T* cs = reinterpret_cast<T*>(p); p += (size_t)D * ts * sizeof(T);
    p = reinterpret_cast<unsigned char*>(((uintptr_t)p + 15) & ~uintptr_t(15));
    uint16_t* perm[2];
    perm[0] = reinterpret_cast<uint16_t*>(p); p += (size_t)ts * 2;
    perm[1] = reinterpret_cast<uint16_t*>(p); p += (size_t)ts * 2;
    p = reinterpret_cast<unsigned char*>(((uintptr_t)p + 15) & ~uintptr_t(15));
    uint32_t* hist_all = reinterpret_cast<uint32_t*>(p);
    cs = as_dyn_shared(cs);
    perm[0] = as_dyn_shared(perm[0]);
    perm[1] = as_dyn_shared(perm[1]);
    hist_all = as_dyn_shared(hist_all);
    uint32_t* hist = hist_all + warp * 256;
    // warp 1's histogram doubles as the mailbox of the root hand-off (it is idle until then)
    volatile int32_t* mbox = reinterpret_cast<volatile int32_t*>(hist_all + 256);
    // stage the task's points with asynchronous copies (all loads in flight at once)
    for (int e = tid; e < n; e += SUB_THREADS) {
        for (int d = 0; d < D; d++) cp_async_elem(&cs[d * ts + e], &src[(int64_t)d * N + tk.start + e]);
        perm[0][e] = (uint16_t)e;
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    pair_sync();
    auto emit = [&](const uint16_t* pm, int st, int len) {
        for (int e = lane; e < len; e += 32) {
            const int qv = pm[st + e];
            for (int d = 0; d < D; d++) buf0[(int64_t)d * N + tk.start + st + e] = cs[d * ts + qv];
            if (pm != perm[0]) perm[0][st + e] = (uint16_t)qv;  // final order collects in perm[0]
        }
    };
    // depth-first, left child first: preorder numbering is the visit order
    int cursor = 0, maxd = 0, sp = 0;
    int st = 0, nn = n, rd = 0, parent_pre = -1;
    uint64_t path = tk.path;
    bool at_root = warp == 0;  // warp 0 is about to process the task's root
    bool work = true;
    int nl_root = 0;
    if (warp != 0) {
        pair_sync();  // root done
        const int nl0 = mbox[0];
        __syncwarp();
        if (nl0 < 0) {
            work = false;  // the root is a leaf
        } else {
            st = nl0;
            nn = n - nl0;
            rd = 1;
            path = tk.path * 2ULL + 1ULL;
            out_nodes += 2 * nl0;
            out_cnt += 2 * nl0;
            stk += 2 * nl0;
        }
    }
    while (work) {
        const int pre = cursor++;
        if (parent_pre >= 0 && lane == 0) out_nodes[parent_pre].a = pre;  // right child index
        maxd = max(maxd, rd);
        int dim = -1, nl = 0;
        double val = 0.0;
        if (nn > c.bucket) {
            const uint16_t* pmn = ((rd & 1) ? perm[1] : perm[0]) + st;
            if constexpr (DT > 0) {
                if (nn <= 64) sub_split_small<T, DT, 2>(cs, pmn, nn, ts, path, c, fyslots, fylocks, dim, val, nl);
                else if (nn <= 128) sub_split_small<T, DT, 4>(cs, pmn, nn, ts, path, c, fyslots, fylocks, dim, val, nl);
                else sub_split<T, DT>(cs, pmn, nn, ts, D, path, c, hist, fyslots, fylocks, dim, val, nl);
            } else {
                sub_split<T, DT>(cs, pmn, nn, ts, D, path, c, hist, fyslots, fylocks, dim, val, nl);
            }
        }
        if (dim < 0) {
            if (lane == 0) {
                out_nodes[pre] = KdNode{0.0, (int32_t)(tk.start + st), -1 - nn};
                out_cnt[pre] = nn;
            }
            emit(perm[rd & 1], st, nn);
            if (at_root) {
                if (lane == 0) mbox[0] = -1;
                pair_sync();
                at_root = false;
            }
            if (sp == 0) break;
            sp--;
            const SubStack e = stk[sp];
            path = e.path;
            parent_pre = e.parent_pre;
            st = (int)(e.packed & 1023u);
            nn = (int)((e.packed >> 10) & 2047u);
            rd = (int)(e.packed >> 21);
            continue;
        }
        // stable partition into the other parity buffer
        const uint16_t* pc = perm[rd & 1];
        uint16_t* pn = perm[(rd + 1) & 1];
        const T* row = cs + dim * ts;
        const T vt = (T)val;  // the split value is a coordinate: comparing in T is exact
        int lrun = 0;
        for (int b = 0; b < nn; b += 128) {  // 4 chunks of 32 per round: loads first, then ballots
            int qv[4];
            bool f[4];
#pragma unroll
            for (int u = 0; u < 4; u++) qv[u] = b + u * 32 + lane < nn ? pc[st + b + u * 32 + lane] : 0;
#pragma unroll
            for (int u = 0; u < 4; u++) f[u] = b + u * 32 + lane < nn && row[qv[u]] < vt;
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int e = b + u * 32 + lane;
                const unsigned bal = __ballot_sync(FULL, f[u]);
                const int lp = __popc(bal & ((1u << lane) - 1));
                if (e < nn) pn[st + (f[u] ? lrun + lp : nl + (e - (lrun + lp)))] = (uint16_t)qv[u];
                lrun += __popc(bal);
            }
        }
        __syncwarp();
        if (at_root) {
            // hand the right child to warp 1 (its index, the size of this warp's part, is patched in below)
            if (lane == 0) {
                out_nodes[pre] = KdNode{val, -1, dim};
                out_cnt[pre] = nn;
                mbox[0] = nl;
            }
            nl_root = nl;
            pair_sync();
            at_root = false;
        } else {
            if (lane == 0) {
                out_nodes[pre] = KdNode{val, -1, dim};
                out_cnt[pre] = nn;
                stk[sp] = SubStack{path * 2ULL + 1ULL, pre,
                                   (uint32_t)(st + nl) | ((uint32_t)(nn - nl) << 10) | ((uint32_t)(rd + 1) << 21)};
            }
            sp++;
        }
        path = path * 2ULL;
        parent_pre = -1;
        nn = nl;
        rd = rd + 1;
        __syncwarp();
    }
    // both parts done: move the right subtree's nodes down behind the left part
    __syncwarp();
    if (!work) cursor = 0;
    if (lane == 0) {
        hist[0] = (uint32_t)cursor;
        hist[1] = (uint32_t)maxd;
        hist[2] = (uint32_t)nl_root;
    }
    pair_sync();
    const int c0 = (int)hist_all[0], c1 = (int)hist_all[256];
    const int md = max((int)hist_all[1], (int)hist_all[257]);
    if (c1 > 0) {
        // the right part was numbered from 0 at scratch index 2*nl (nl = the root's left count)
        const int nl0 = (int)hist_all[2];
        KdNode* base_nodes = scratch + 2 * tk.start;
        int32_t* base_cnt = scnt + 2 * tk.start;
        const KdNode* rs = base_nodes + 2 * nl0;
        const int32_t* rc = base_cnt + 2 * nl0;
        for (int b = 0; b < c1; b += SUB_THREADS) {  // destination <= source: ascending chunks, read before write
            const int i = b + tid;
            KdNode nd = KdNode{0.0, 0, 0};
            int32_t cn = 0;
            if (i < c1) {
                nd = rs[i];
                cn = rc[i];
                if (nd.db >= 0) nd.a += c0;
            }
            pair_sync();
            if (i < c1) {
                base_nodes[c0 + i] = nd;
                base_cnt[c0 + i] = cn;
            }
            pair_sync();
        }
        if (tid == 0) base_nodes[0].a = c0;
    }
    // row ids in the final order; the source may alias the output, so read all before writing
    int32_t rid[MAXS / SUB_THREADS];
#pragma unroll
    for (int k2 = 0; k2 < MAXS / SUB_THREADS; k2++) {
        const int e = k2 * SUB_THREADS + tid;
        if (e < n) rid[k2] = isrc ? isrc[tk.start + perm[0][e]] : (int32_t)(tk.start + perm[0][e]);
    }
    pair_sync();
#pragma unroll
    for (int k2 = 0; k2 < MAXS / SUB_THREADS; k2++) {
        const int e = k2 * SUB_THREADS + tid;
        if (e < n) idx0[tk.start + e] = rid[k2];
    }
    if (tid == 0) {
        task_nodes[task] = c0 + c1;
        task_depth[task] = tk.depth + md;
    }
}

// ============================================================================
// preorder stitch of the breadth-first top and the subtree tasks
// ============================================================================
__device__ __forceinline__ int child_nodes(const TopStore& ts, const int32_t* task_nodes, int s) {
    return ts.kind[s] == TS_TASK ? task_nodes[ts.task[s]] : ts.nodes[s];
}

static __global__ void k_top_count(const LNode* lv, int K, TopStore ts, const int32_t* task_nodes) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const int s = lv[i].slot;
    if (ts.kind[s] != TS_INTERIOR) return;
    ts.nodes[s] = 1 + child_nodes(ts, task_nodes, ts.left[s]) + child_nodes(ts, task_nodes, ts.right[s]);
}

static __global__ void k_top_pre(const LNode* lv, int K, TopStore ts, const int32_t* task_nodes, int32_t* task_base,
                          KdNode* nodes, int32_t* ncount) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= K) return;
    const int s = lv[i].slot;
    if (ts.kind[s] != TS_INTERIOR) return;
    const int p = ts.pre[s];
    const int l = ts.left[s], r = ts.right[s];
    const int pl = p + 1, pr = p + 1 + child_nodes(ts, task_nodes, l);
    ts.pre[l] = pl;
    ts.pre[r] = pr;
    if (ts.kind[l] == TS_TASK) task_base[ts.task[l]] = pl;
    if (ts.kind[r] == TS_TASK) task_base[ts.task[r]] = pr;
    nodes[p] = KdNode{ts.val[s], pr, ts.dim[s]};
    ncount[p] = ts.npts[s];
}

// small trees: the whole stitch in one CTA (counts bottom-up, then preorder top-down, one
// barrier per level) instead of two launches per level -- a 1M-point build spends 10 % of
// its time in those launches
constexpr int TOP_FUSED_LEVELS = 48;
constexpr int TOP_FUSED_NODES = 16384;
struct LevelList {
    const LNode* lv[TOP_FUSED_LEVELS];
    int k[TOP_FUSED_LEVELS];
    int count;
};
static __global__ void __launch_bounds__(1024) k_top_count_all(LevelList L, TopStore ts, const int32_t* task_nodes) {
    for (int l = L.count - 1; l >= 0; l--) {
        for (int i = threadIdx.x; i < L.k[l]; i += blockDim.x) {
            const int s = L.lv[l][i].slot;
            if (ts.kind[s] != TS_INTERIOR) continue;
            ts.nodes[s] = 1 + child_nodes(ts, task_nodes, ts.left[s]) + child_nodes(ts, task_nodes, ts.right[s]);
        }
        __syncthreads();
    }
}
static __global__ void __launch_bounds__(1024) k_top_pre_all(LevelList L, TopStore ts, const int32_t* task_nodes,
                                                             int32_t* task_base, KdNode* nodes, int32_t* ncount) {
    for (int l = 0; l < L.count; l++) {
        for (int i = threadIdx.x; i < L.k[l]; i += blockDim.x) {
            const int s = L.lv[l][i].slot;
            if (ts.kind[s] != TS_INTERIOR) continue;
            const int p = ts.pre[s];
            const int lc = ts.left[s], rc = ts.right[s];
            const int pl = p + 1, pr = p + 1 + child_nodes(ts, task_nodes, lc);
            ts.pre[lc] = pl;
            ts.pre[rc] = pr;
            if (ts.kind[lc] == TS_TASK) task_base[ts.task[lc]] = pl;
            if (ts.kind[rc] == TS_TASK) task_base[ts.task[rc]] = pr;
            nodes[p] = KdNode{ts.val[s], pr, ts.dim[s]};
            ncount[p] = ts.npts[s];
        }
        __syncthreads();
    }
}

static __global__ void k_relocate(const Task* tasks, const int32_t* task_nodes, const int32_t* task_base,
                           const KdNode* scratch, const int32_t* scnt, KdNode* nodes, int32_t* ncount) {
    const Task tk = tasks[blockIdx.x];
    const int cnt = task_nodes[blockIdx.x];
    const int base = task_base[blockIdx.x];
    const KdNode* src = scratch + 2 * tk.start;
    const int32_t* sc = scnt + 2 * tk.start;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
        KdNode nd = src[i];
        if (nd.db >= 0) nd.a += base;
        nodes[base + i] = nd;
        ncount[base + i] = sc[i];
    }
}

static __global__ void k_gather_ids(const uint64_t* __restrict__ ids_in, const int32_t* __restrict__ perm,
                             uint64_t* __restrict__ ids_out, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) ids_out[i] = ids_in ? ids_in[perm[i]] : (uint64_t)perm[i];
}


// ============================================================================
// host orchestration
// ============================================================================
static bool trace_alloc() {
    static const bool v = std::getenv("KDB_TRACE_ALLOC") != nullptr;
    return v;
}

template <typename X>
static X* palloc(size_t count, cudaStream_t st) {  // pool: buffers that outlive the build
    void* p = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    KD_CUDA(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(X), st));
    if (trace_alloc()) {
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (ms > 0.5) fprintf(stderr, "[kdb] slow cudaMallocAsync %.3f ms for %zu bytes\n", ms, count * sizeof(X));
    }
    return static_cast<X*>(p);
}
template <typename X>
static X* dalloc(size_t count, cudaStream_t st) {  // build scratch
    if (t_arena) return static_cast<X*>(t_arena->alloc(std::max<size_t>(count, 1) * sizeof(X)));
    return palloc<X>(count, st);
}
static void dfree(void* p, cudaStream_t st) {
    if (p && !(t_arena && t_arena->owns(p))) cudaFreeAsync(p, st);
}

// keep freed stream-ordered allocations in the pool across the per-level host
// synchronisations (the default release threshold of 0 returns them to the
// driver at every sync and re-maps them on the next level)
// persistent pinned words for the per-level counter read-back (page-locking per build costs ms)
// (one per host thread: concurrent builds from several rank threads must not share it)
static unsigned long long* pinned_counters(int) {
    static thread_local unsigned long long* p = nullptr;  // [0] next level, [1] tasks|slow, [2] max node
    if (!p) KD_CUDA(cudaMallocHost(&p, 4 * sizeof(unsigned long long)));
    return p;
}

uint32_t* fy_slots(int device, cudaStream_t st);  // persistent per-device scratch (kd_build_f32.cu)
#ifdef KD_BUILD_COMMON
static std::mutex g_init_mu;

// persistent per-device scratch for the rare exact-variance path of k_subtree
uint32_t* fy_slots(int device, cudaStream_t st) {
    static uint32_t* slots[64] = {nullptr};
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (!slots[device]) {
        const size_t words = (size_t)FY_SLOTS * 2 * MAXS + FY_SLOTS;
        KD_CUDA(cudaMalloc(&slots[device], words * 4));
        KD_CUDA(cudaMemsetAsync(slots[device] + (size_t)FY_SLOTS * 2 * MAXS, 0, FY_SLOTS * 4, st));
    }
    return slots[device];
}

static std::vector<Arena*> g_arenas[64];
static std::mutex g_arena_mu;  // never held across a CUDA call (released from stream host callbacks)
Arena* arena_acquire(int device) {
    std::lock_guard<std::mutex> lk(g_arena_mu);
    std::vector<Arena*>& fl = g_arenas[device & 63];
    Arena* a = nullptr;
    if (!fl.empty()) {
        a = fl.back();
        fl.pop_back();
    } else {
        a = new Arena();
        a->device = device;
    }
    a->reset();
    return a;
}
void arena_release(Arena* a) {
    std::lock_guard<std::mutex> lk(g_arena_mu);
    g_arenas[a->device & 63].push_back(a);
}

void retain_pool(int device) {
    static bool done[64] = {false};
    std::lock_guard<std::mutex> lk(g_init_mu);
    if (device < 0 || device >= 64 || done[device]) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = ~0ULL;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done[device] = true;
}

#endif

struct HostTrace {
    bool on = std::getenv("KDB_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(const char* what, int a = -1) {
        if (!on) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        fprintf(stderr, "[kdb] %9.3f ms  %s %d\n", ms, what, a);
    }
    void sync_mark(cudaStream_t st, const char* what, int a = -1) {  // tracing only: waits for the stream
        if (!on) return;
        cudaStreamSynchronize(st);
        mark(what, a);
    }
};

template <typename T>
void build_tree(const T* d_in, const uint64_t* d_ids, int64_t n, int dims, const BuildCfg& cfg, cudaStream_t st,
                KdTreeDev* out, BuildStats* stats) {
    HostTrace tr;
    tr.mark("enter");
    cudaEvent_t e0, e1, e_top, e_sub;
    KD_CUDA(cudaEventCreate(&e0));
    KD_CUDA(cudaEventCreate(&e1));
    KD_CUDA(cudaEventCreate(&e_top));
    KD_CUDA(cudaEventCreate(&e_sub));
    KD_CUDA(cudaEventRecord(e0, st));
    out->dims = dims;
    out->n = n;
    out->dtype = sizeof(T) == 4 ? DT_F32 : DT_F64;
    KD_CUDA(cudaGetDevice(&out->device));
    retain_pool(out->device);
    if (n == 0) {
        out->n_nodes = 0; out->n_leaves = 0; out->depth = 0;
        out->nodes = palloc<KdNode>(1, st);
        out->node_count = palloc<int32_t>(1, st);
        out->coords = palloc<T>(1, st);
        out->ids = palloc<uint64_t>(1, st);
        out->perm = palloc<int32_t>(1, st);
        KD_CUDA(cudaStreamSynchronize(st));
        cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(e_top); cudaEventDestroy(e_sub);
        return;
    }
    DevCtx c;
    c.dims = dims;
    c.N = n;
    c.bucket = cfg.bucket;
    c.ms = cfg.msample;
    c.vs = cfg.vsample;
    c.seed = cfg.seed;
    c.ts = (int)std::min<int64_t>({(int64_t)MAXS, cfg.msample, cfg.vsample});
    // shared-memory capacity caps the subtree size for wide / f64 points
    int dev_smem = 0;
    KD_CUDA(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, out->device));
    while (c.ts > 32 && sub_smem_bytes(c.ts, dims, sizeof(T)) > (size_t)dev_smem) c.ts /= 2;
    c.ts = std::max<int>(c.ts, 1);

    ArenaScope arena(out->device);
    // buf[0] / idx[0] end as the tree's packed coordinates / row ids
    T* buf[2] = {palloc<T>((size_t)dims * n, st), dalloc<T>((size_t)dims * n, st)};
    int32_t* idx[2] = {palloc<int32_t>(n, st), dalloc<int32_t>(n, st)};

    // the bulk-copy (TMA) tile loads start at the 16-byte boundary below a tile: a caller's buffer
    // that is not 16-byte aligned (a view into a larger tensor) is first copied into build scratch
    if (reinterpret_cast<uintptr_t>(d_in) & 15) {
        T* aligned = dalloc<T>((size_t)dims * n, st);
        KD_CUDA(cudaMemcpyAsync(aligned, d_in, sizeof(T) * (size_t)dims * n, cudaMemcpyDeviceToDevice, st));
        d_in = aligned;
    }

    // top store (grown per level)
    size_t ts_cap = 1024;
    TopStore ts{};
    auto ts_alloc = [&](size_t cap) {
        TopStore t2{};
        t2.dim = dalloc<int32_t>(cap, st); t2.val = dalloc<double>(cap, st);
        t2.left = dalloc<int32_t>(cap, st); t2.right = dalloc<int32_t>(cap, st);
        t2.npts = dalloc<int32_t>(cap, st); t2.kind = dalloc<int32_t>(cap, st);
        t2.task = dalloc<int32_t>(cap, st); t2.nodes = dalloc<int32_t>(cap, st);
        t2.pre = dalloc<int32_t>(cap, st);
        return t2;
    };
    auto ts_free = [&](TopStore& t2) {
        dfree(t2.dim, st); dfree(t2.val, st); dfree(t2.left, st); dfree(t2.right, st); dfree(t2.npts, st);
        dfree(t2.kind, st); dfree(t2.task, st); dfree(t2.nodes, st); dfree(t2.pre, st);
    };
    ts = ts_alloc(ts_cap);
    size_t ts_used = 1;
    // tasks: at most one per point range; bounded by 2 * (#top nodes) + 1 -> grow with the store
    size_t task_cap = 1024;
    Task* tasks = dalloc<Task>(task_cap, st);
    // level counters in one block (one clear and one read-back per level):
    //   [0] next level's packed (node count << 32 | tiles), [1] max child size (low) | slow nodes (high),
    //   [2] subtree task count (cumulative over levels)
    unsigned long long* ctr = dalloc<unsigned long long>(3, st);
    KD_CUDA(cudaMemsetAsync(ctr, 0, 3 * sizeof(unsigned long long), st));
    unsigned long long* next_ctr = ctr;
    int* next_max = reinterpret_cast<int*>(ctr + 1);
    int* slow_count = next_max + 1;
    int* task_ctr = reinterpret_cast<int*>(ctr + 2);
    unsigned long long* h_ctr = nullptr;
    h_ctr = pinned_counters(out->device);

    std::vector<LNode*> levels;
    std::vector<int> level_k;
    int K = 0;
    uint32_t tiles = 0;
    {
        // root
        const int32_t kind_root = n > c.ts ? TS_INTERIOR : TS_TASK;
        KD_CUDA(cudaMemcpyAsync(ts.kind, &kind_root, sizeof(int32_t), cudaMemcpyHostToDevice, st));
        const int32_t zero = 0;
        KD_CUDA(cudaMemcpyAsync(ts.pre, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, st));
        if (n > c.ts) {
            LNode root{0, (int32_t)n, 0, 1ULL, 0, 0};
            LNode* l0 = dalloc<LNode>(1, st);
            KD_CUDA(cudaMemcpyAsync(l0, &root, sizeof(LNode), cudaMemcpyHostToDevice, st));
            levels.push_back(l0);
            K = 1;
            tiles = (uint32_t)((n + TILE - 1) / TILE);
        } else {
            Task t0{0, (int32_t)n, 0, 1ULL, 0, 2, 0, 0};  // reads the input directly
            KD_CUDA(cudaMemcpyAsync(tasks, &t0, sizeof(Task), cudaMemcpyHostToDevice, st));
            const int one = 1;
            KD_CUDA(cudaMemcpyAsync(task_ctr, &one, sizeof(int), cudaMemcpyHostToDevice, st));
            const int32_t z = 0;
            KD_CUDA(cudaMemcpyAsync(ts.task, &z, sizeof(int32_t), cudaMemcpyHostToDevice, st));
        }
    }
    int ntasks_known = K == 0 ? 1 : 0;
    {
    }
    const size_t sample_smem32 = (size_t)SAMPLE_WARPS * (std::max<size_t>(4 * MAXS, 2 * FYD_MAX) + MAXS * (4 + 2));
    const size_t sample_smem64 = (size_t)SAMPLE_WARPS * (std::max<size_t>(8 * MAXS, 2 * FYD_MAX) + MAXS * (4 + 2));
    KD_CUDA(cudaFuncSetAttribute(k_sample<T, 3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sample_smem32));
    KD_CUDA(cudaFuncSetAttribute(k_sample<T, 0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sample_smem32));
    KD_CUDA(cudaFuncSetAttribute(k_sample<T, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sample_smem64));
    KD_CUDA(cudaFuncSetAttribute(k_sample<T, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sample_smem64));
    // levels with at most this many nodes choose splits with a CTA per node (KDB_SAMPLE_CTA_K overrides)
    static const int sample_cta_max = [] {
        const char* e = std::getenv("KDB_SAMPLE_CTA_K");
        return e ? atoi(e) : 1024;
    }();
    uint32_t scatter_grid = 0, hist_grid = 0;  // resident CTAs of the persistent scatter / histogram
    uint32_t scatter_tma_grid = 0;
    size_t scatter_tma_smem = 0;
    static const bool scatter_tma = std::getenv("KDB_NO_SCATTER_TMA") == nullptr;
    {
        int sms = 148, per = 0;
        KD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, out->device));
        KD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_scatter<T, 3, 8>, TILE_THREADS, 0));
        scatter_grid = (uint32_t)sms * (uint32_t)std::max(per, 1);
        if (dims == 2 || dims == 3) {  // TMA-fed variant: two shared-memory stages per CTA
            const size_t sb = 2 * (dims == 2 ? scat_stage_bytes<T, 2>() : scat_stage_bytes<T, 3>());
            if (dims == 2) {
                KD_CUDA(cudaFuncSetAttribute(k_scatter_tma<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
                KD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_scatter_tma<T, 2>, TILE_THREADS, sb));
            } else {
                KD_CUDA(cudaFuncSetAttribute(k_scatter_tma<T, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sb));
                KD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_scatter_tma<T, 3>, TILE_THREADS, sb));
            }
            scatter_tma_grid = (uint32_t)sms * (uint32_t)std::max(per, 1);
            scatter_tma_smem = sb;
        }
        KD_CUDA(cudaFuncSetAttribute(k_hist<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(2 * HIST_SLOT<T> * sizeof(T))));
        KD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_hist<T>, TILE_THREADS, 2 * HIST_SLOT<T> * sizeof(T)));
        hist_grid = (uint32_t)sms * (uint32_t)std::max(per, 1);
    }
    int par = 0;  // buffer holding the current level's points
    int64_t slow_total = 0;
    int64_t max_node = n;  // largest node of the current level (read back with the level counters)
    bool at_input = true;  // the first level reads the caller's points directly (row ids = positions)
    // per-level scratch, allocated once at bounds that hold for every level: a level's
    // nodes all exceed ts points, so K <= n / (ts + 1) + 1, and its tiles <= n / TILE + K
    const size_t kmax = (size_t)(n / (c.ts + 1)) + 2;
    const size_t tmax = (size_t)(n / TILE) + kmax + 1;
    Split* split = dalloc<Split>(kmax, st);
    T* wb = dalloc<T>(kmax * WIN, st);
    uint32_t* wf = dalloc<uint32_t>(kmax * WIN, st);
    int* slow_list = dalloc<int>(kmax, st);
    uint32_t* tile_left = dalloc<uint32_t>(tmax * SUB + 1, st);
    uint32_t* tile_loff = dalloc<uint32_t>(tmax * SUB + 1, st);
    int32_t* tmap = dalloc<int32_t>(tmax, st);
    uint16_t* hrow = dalloc<uint16_t>(tmax * SUB * WIN, st);
    uint32_t* hL = dalloc<uint32_t>(tmax * SUB, st);
    TileInfo* tinfo = dalloc<TileInfo>(tmax, st);
    HalfMeta* hmeta = dalloc<HalfMeta>(tmax * SUB, st);
    size_t scan_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, tile_left, tile_loff, (int)(tmax * SUB), st);
    void* scan_tmp = dalloc<unsigned char>(scan_bytes, st);
    while (K > 0) {
        LNode* lv = levels.back();
        if ((size_t)K > kmax || (size_t)tiles > tmax) throw CudaError{"level exceeds the preallocated bounds"};
        const T* lsrc = at_input ? d_in : buf[par];
        const int32_t* lidx = at_input ? nullptr : idx[par];
        const bool big_levels = max_node > (int64_t(1) << 22);
        // capacity: children slots and tasks
        if (ts_used + 2 * (size_t)K + 1 > ts_cap) {
            size_t nc = std::max(ts_cap * 2, ts_used + 2 * (size_t)K + 1);
            TopStore t2 = ts_alloc(nc);
            auto cp = [&](void* d, void* s, size_t b) { KD_CUDA(cudaMemcpyAsync(d, s, b, cudaMemcpyDeviceToDevice, st)); };
            cp(t2.dim, ts.dim, ts_used * 4); cp(t2.val, ts.val, ts_used * 8); cp(t2.left, ts.left, ts_used * 4);
            cp(t2.right, ts.right, ts_used * 4); cp(t2.npts, ts.npts, ts_used * 4); cp(t2.kind, ts.kind, ts_used * 4);
            cp(t2.task, ts.task, ts_used * 4); cp(t2.pre, ts.pre, ts_used * 4);
            ts_free(ts);
            ts = t2;
            ts_cap = nc;
        }
        if ((size_t)ntasks_known + 2 * (size_t)K + 1 > task_cap) {
            size_t nc = std::max(task_cap * 2, (size_t)ntasks_known + 2 * (size_t)K + 1);
            Task* t2 = dalloc<Task>(nc, st);
            KD_CUDA(cudaMemcpyAsync(t2, tasks, sizeof(Task) * ntasks_known, cudaMemcpyDeviceToDevice, st));
            dfree(tasks, st);
            tasks = t2;
            task_cap = nc;
        }
        KD_CUDA(cudaMemsetAsync(ctr, 0, 2 * sizeof(unsigned long long), st));  // next, max child, slow nodes
        if (K <= sample_cta_max) {
            if (dims == 3) k_sample_cta<T, 3><<<K, CTA_S, 0, st>>>(lsrc, lv, c, split, wb, wf);
            else k_sample_cta<T, 0><<<K, CTA_S, 0, st>>>(lsrc, lv, c, split, wb, wf);
        } else {
            const unsigned sg = (unsigned)((K + SAMPLE_WARPS - 1) / SAMPLE_WARPS);
            if (dims == 3) {
                k_sample<T, 3, false><<<sg, SAMPLE_WARPS * 32, sample_smem32, st>>>(lsrc, lv, K, c, split, wb, wf);
                if (big_levels) k_sample<T, 3, true><<<sg, SAMPLE_WARPS * 32, sample_smem64, st>>>(lsrc, lv, K, c, split, wb, wf);
            } else {
                k_sample<T, 0, false><<<sg, SAMPLE_WARPS * 32, sample_smem32, st>>>(lsrc, lv, K, c, split, wb, wf);
                if (big_levels) k_sample<T, 0, true><<<sg, SAMPLE_WARPS * 32, sample_smem64, st>>>(lsrc, lv, K, c, split, wb, wf);
            }
        }
        k_tile_info<<<(tiles + 255) / 256, 256, 0, st>>>(lv, K, tmap, split, tiles, c.N, tinfo);
        k_hist<T><<<std::min<uint32_t>(tiles, hist_grid), TILE_THREADS, 2 * HIST_SLOT<T> * sizeof(T), st>>>(lsrc, tinfo, tiles, split, wb, wf, hrow,
                                                                                  hL);
        k_select<T><<<(K + 3) / 4, 128, 0, st>>>(lv, K, split, wb, wf, slow_list, slow_count);
        k_slow<T><<<std::min(K, 1024), SLOW_THREADS, 0, st>>>(lsrc, lv, c, split, slow_list, slow_count);
        k_tile_left<T><<<(tiles * SUB + 7) / 8, 256, 0, st>>>(lsrc, lv, tmap, c, split, hrow, hL, tiles * SUB, tile_left,
                                                                hmeta);
        {
            size_t need = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, need, tile_left, tile_loff, (int)(tiles * SUB), st);
            if (need > scan_bytes) {
                dfree(scan_tmp, st);
                scan_tmp = dalloc<unsigned char>(need, st);
                scan_bytes = need;
            }
            cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, tile_left, tile_loff, (int)(tiles * SUB), st);
        }
#define KD_SCATTER(DTV, CHV)                                                                                   \
    k_scatter<T, DTV, CHV><<<std::min<uint32_t>(tiles * SUB, scatter_grid), TILE_THREADS, 0, st>>>(                  \
        lsrc, lidx, buf[1 - par], idx[1 - par], hmeta, c, tile_loff, tiles * SUB)
#define KD_SCATTER_TMA(DTV)                                                                                     \
    k_scatter_tma<T, DTV><<<std::min<uint32_t>(tiles * SUB, scatter_tma_grid), TILE_THREADS, scatter_tma_smem, st>>>( \
        lsrc, lidx, buf[1 - par], idx[1 - par], hmeta, c, tile_loff, tiles * SUB)
        switch (dims) {
            case 1: KD_SCATTER(1, 8); break;
            case 2: if (scatter_tma) KD_SCATTER_TMA(2); else KD_SCATTER(2, 8); break;
            case 3: if (scatter_tma) KD_SCATTER_TMA(3); else KD_SCATTER(3, 8); break;
            case 4: KD_SCATTER(4, 8); break;
            default: KD_SCATTER(0, 2); break;
        }
#undef KD_SCATTER
#undef KD_SCATTER_TMA
        LNode* next = dalloc<LNode>(2 * (size_t)K, st);
        k_children<<<(K + 255) / 256, 256, 0, st>>>(lv, K, split, c, 1 - par, at_input ? 2 : par, (int)ts_used, ts, next, next_ctr,
                                                    tasks, task_ctr, next_max);
        KD_CUDA(cudaGetLastError());
        KD_CUDA(cudaMemcpyAsync(h_ctr, ctr, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        KD_CUDA(cudaStreamSynchronize(st));
        tr.mark("level done", (int)levels.size());
        slow_total += (int)(h_ctr[1] >> 32);
        ntasks_known = (int)(h_ctr[2] & 0xFFFFFFFFULL);
        level_k.push_back(K);
        ts_used += 2 * (size_t)K;
        K = (int)(h_ctr[0] >> 32);
        tiles = (uint32_t)(h_ctr[0] & 0xFFFFFFFFULL);
        max_node = (int64_t)(int32_t)(h_ctr[1] & 0xFFFFFFFFULL);
        par = 1 - par;
        at_input = false;
        if (K > 0) levels.push_back(next);
        else dfree(next, st);
    }
    dfree(split, st); dfree(wb, st); dfree(wf, st); dfree(slow_list, st); dfree(tile_left, st); dfree(tile_loff, st);
    dfree(tmap, st); dfree(hrow, st); dfree(hL, st); dfree(tinfo, st); dfree(hmeta, st); dfree(scan_tmp, st);
    tr.mark("top phase done");
    const int ntasks = ntasks_known > 0 ? ntasks_known : 1;
    // subtree phase
    KD_CUDA(cudaEventRecord(e_top, st));
    tr.sync_mark(st, "top scratch freed");
    KdNode* scratch = dalloc<KdNode>(2 * (size_t)n + 2, st);
    int32_t* scnt = dalloc<int32_t>(2 * (size_t)n + 2, st);
    int32_t* task_nodes = dalloc<int32_t>(ntasks, st);
    int32_t* task_depth = dalloc<int32_t>(ntasks, st);
    int32_t* task_base = dalloc<int32_t>(ntasks, st);
    const size_t sub_smem = sub_smem_bytes(c.ts, dims, sizeof(T));
    SubStack* sstack = dalloc<SubStack>(2 * (size_t)n + 2, st);
    uint32_t* fyslots = fy_slots(out->device, st);
    tr.sync_mark(st, "subtree scratch allocated");
    int* fylocks = reinterpret_cast<int*>(fyslots + (size_t)FY_SLOTS * 2 * MAXS);
    if (dims == 3) {
        KD_CUDA(cudaFuncSetAttribute(k_subtree<T, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sub_smem));
        k_subtree<T, 3><<<ntasks, SUB_THREADS, sub_smem, st>>>(tasks, buf[0], buf[1], d_in, idx[0], idx[1], c, scratch, scnt, sstack,
                                                      fyslots, fylocks, task_nodes, task_depth);
    } else {
        KD_CUDA(cudaFuncSetAttribute(k_subtree<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sub_smem));
        k_subtree<T, 0><<<ntasks, SUB_THREADS, sub_smem, st>>>(tasks, buf[0], buf[1], d_in, idx[0], idx[1], c, scratch, scnt, sstack,
                                                      fyslots, fylocks, task_nodes, task_depth);
    }
    KD_CUDA(cudaGetLastError());
    KD_CUDA(cudaEventRecord(e_sub, st));
    tr.sync_mark(st, "k_subtree done", ntasks);
    // top counts bottom-up, preorder top-down
    size_t top_nodes = 0;
    for (int kk : level_k) top_nodes += (size_t)kk;
    const bool top_fused = levels.size() <= (size_t)TOP_FUSED_LEVELS && top_nodes <= (size_t)TOP_FUSED_NODES;
    LevelList ll;
    ll.count = 0;
    if (top_fused) {
        for (size_t L = 0; L < levels.size(); L++) { ll.lv[L] = levels[L]; ll.k[L] = level_k[L]; }
        ll.count = (int)levels.size();
        if (ll.count) k_top_count_all<<<1, 1024, 0, st>>>(ll, ts, task_nodes);
    } else {
        for (int L = (int)levels.size() - 1; L >= 0; L--)
            k_top_count<<<(level_k[L] + 255) / 256, 256, 0, st>>>(levels[L], level_k[L], ts, task_nodes);
    }
    int32_t total_nodes = 0;
    {
        int32_t root_kind = 0;
        KD_CUDA(cudaMemcpyAsync(&root_kind, ts.kind, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        KD_CUDA(cudaStreamSynchronize(st));
        const int32_t* src = root_kind == TS_TASK ? task_nodes : ts.nodes;
        KD_CUDA(cudaMemcpyAsync(&total_nodes, src, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        if (root_kind == TS_TASK) KD_CUDA(cudaMemsetAsync(task_base, 0, sizeof(int32_t), st));
        KD_CUDA(cudaStreamSynchronize(st));
    }
    KdNode* nodes = palloc<KdNode>(total_nodes, st);
    int32_t* ncount = palloc<int32_t>(total_nodes, st);
    if (top_fused) {
        if (ll.count) k_top_pre_all<<<1, 1024, 0, st>>>(ll, ts, task_nodes, task_base, nodes, ncount);
    } else {
        for (size_t L = 0; L < levels.size(); L++)
            k_top_pre<<<(level_k[L] + 255) / 256, 256, 0, st>>>(levels[L], level_k[L], ts, task_nodes, task_base, nodes,
                                                                ncount);
    }
    tr.sync_mark(st, "preorder done");
    k_relocate<<<ntasks, 256, 0, st>>>(tasks, task_nodes, task_base, scratch, scnt, nodes, ncount);
    tr.sync_mark(st, "relocate done");
    uint64_t* ids_out = palloc<uint64_t>(n, st);
    k_gather_ids<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_ids, idx[0], ids_out, n);
    KD_CUDA(cudaGetLastError());
    // depth = max(task depths, top levels)
    std::vector<int32_t> hdepth(ntasks);
    KD_CUDA(cudaMemcpyAsync(hdepth.data(), task_depth, sizeof(int32_t) * ntasks, cudaMemcpyDeviceToHost, st));
    KD_CUDA(cudaEventRecord(e1, st));
    KD_CUDA(cudaStreamSynchronize(st));
    tr.mark("finalize done");
    int64_t depth = 0;
    for (int i = 0; i < ntasks_known; i++) depth = std::max<int64_t>(depth, hdepth[i]);
    out->n_nodes = total_nodes;
    out->n_leaves = ((int64_t)total_nodes + 1) / 2;  // full binary tree: every interior node has two children
    out->depth = depth;
    out->nodes = nodes;
    out->node_count = ncount;
    out->coords = buf[0];
    out->ids = ids_out;
    out->perm = idx[0];
    if (stats) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        stats->ms_total = ms;
        float a = 0, b = 0, c = 0;
        cudaEventElapsedTime(&a, e0, e_top);
        cudaEventElapsedTime(&b, e_top, e_sub);
        cudaEventElapsedTime(&c, e_sub, e1);
        stats->ms_levels = a;
        stats->ms_subtree = b;
        stats->ms_finish = c;
        stats->levels = (int)levels.size();
        stats->tasks = ntasks_known;
        stats->slow_nodes = slow_total;
    }
    // release scratch
    dfree(buf[1], st); dfree(idx[1], st);
    for (auto l : levels) dfree(l, st);
    ts_free(ts);
    dfree(tasks, st); dfree(ctr, st);
    dfree(scratch, st); dfree(scnt, st); dfree(sstack, st); dfree(task_nodes, st); dfree(task_depth, st); dfree(task_base, st);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e_top);
    cudaEventDestroy(e_sub);
    KD_CUDA(cudaStreamSynchronize(st));
    tr.mark("exit");
}

#ifdef KD_BUILD_COMMON
// every tree buffer comes from the device's stream-ordered pool (cudaMallocAsync); freeing
// with cudaFreeAsync returns it to the pool.  (cudaFree would hand the physical pages
// back to the driver, and the next build would pay for re-mapping them: measured
// 10-200 ms stalls in the first breadth-first level of a 256M-point build.)
void free_tree(KdTreeDev* t) {
    if (!t) return;
    for (void* p : {(void*)t->nodes, (void*)t->node_count, t->coords, (void*)t->ids, (void*)t->perm,
                    (void*)t->qnodes})
        if (p) cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
    t->qnodes = nullptr;
    t->nodes = nullptr; t->node_count = nullptr; t->coords = nullptr; t->ids = nullptr; t->perm = nullptr;
}

#endif

}  // namespace kdb
