// kd_query.cu -- exact k-nearest-neighbour search (Algorithm 1, local_query.py:72-172).
//
// 2-D / 3-D, k(+1) <= 32 (the BASELINE configs): queries are ordered by 32-bit Morton keys
// (k_qbox, k_morton, radix sort), then two passes --
//   k_knn_home     thread per query: descent to the home leaf, an upper bound on the k-th
//                  distance from that bucket (fp32, rounded up, for float trees) and the first
//                  path node whose far child can matter;
//   k_knn_persist  persistent warps, one query per lane from a warp-local pool of the sorted
//                  order: explicit stack of far children with per-dimension fp32 box offsets,
//                  chunked bucket scans with deferred insertion into a register top-k list.
// D >= 4: k_knn_wq (warp per query).  k > 32: k_knn (thread per query, the reference's heap).
// Any depth / the reference's own walk and counters: kd_walk.cu.
// Common to all of them:
//   * pruning bound = sum of squared offsets evaluated in fp32 with round-toward-zero steps,
//     provably <= the binary64 distance of every point in the box (monotone rounding), so
//     pruning never loses a neighbour;
//   * leaf scan in binary64 with the reference's exact operation order (core.py:199-228:
//     ascending dimension, no FMA) -> bit-identical keys;
//   * tie semantics of the brute-force oracle (pkg/tests/conftest.py:8-18): admit d < radius
//     while under-full, replace on lexicographic (d, id) when full, prune only when
//     bound > k-th distance.  (The reference prunes at bound >= r' and can lose an exact tie
//     with a smaller id: SURVEY §8(a) Q5; KD_KNN_REFERENCE reproduces that walk.)
#include <cub/cub.cuh>

#include <algorithm>
#include <map>
#include <mutex>

#include "kd_arena.cuh"
#include "kd_common.cuh"
#include "kd_query.cuh"
#include "kd_topk.cuh"
#include "kd_tree.cuh"
#include "kd_warp.cuh"

namespace kdb {


// traversal stack capacity of the per-query kernels: a depth-first walk that pushes
// only far children holds at most one entry per tree level, and kd_knn refuses trees
// deeper than KNN_MAX_DEPTH = QCAP - 3 for these kernels (KD_EUNSUPPORTED), so a
// push can never overflow; the `sp < QCAP` terms in the push conditions are
// therefore always true (they stay: without them nvcc schedules the persistent
// kernel's push ~5 % slower on C2/C3, measured)
#ifndef KD_KNN_CTAS
#define KD_KNN_CTAS 7
#endif
#ifndef KD_HOME_F32
#define KD_HOME_F32 1
#endif
constexpr int QCAP = 40;
constexpr int KNN_MORTON_BITS = 32;  // Morton key bits of the 3-D query order
// the fp32 pre-filter costs the persistent kernel more in registers/occupancy than it saves in 2-3 D
// (measured 34 vs 44 ms on C2); in higher dimensions the binary64 leaf scan dominates and it pays off
template <int DT>
constexpr bool kPersistF32Filter = (DT == 0);

template <int DT>
struct Dims {
    static constexpr int cap = DT > 0 ? DT : 16;
};

template <typename T, int DT, int KM>
__global__ void __launch_bounds__(128)
k_knn(const KdNode* __restrict__ nodes, int64_t n_nodes, const T* __restrict__ coords,
      const uint64_t* __restrict__ ids, int64_t n, int dims_rt, const double* __restrict__ queries,
      const int32_t* __restrict__ order, int64_t nq, int k, const double* __restrict__ radii,
      const uint64_t* __restrict__ excl, double* __restrict__ out_d, uint64_t* __restrict__ out_i,
      int64_t* __restrict__ out_c, int64_t* __restrict__ out_ctr, double* __restrict__ heap_d,
      uint64_t* __restrict__ heap_i) {
    constexpr int DC = Dims<DT>::cap;
    const int D = DT > 0 ? DT : dims_rt;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nq) return;
    const int64_t qi = order ? (int64_t)order[t] : t;
    double q[DC];
#pragma unroll
    for (int d = 0; d < DC; d++) q[d] = d < D ? queries[qi * D + d] : 0.0;
    const double radius = radii ? radii[qi] : INFINITY;
    const uint64_t ex = excl ? excl[qi] : ~0ULL;
    const bool has_ex = excl != nullptr;
    int64_t c0 = 0, c1 = 0, c2 = 0;

    // top-k state
    double bd[KM > 0 ? KM : 1];
    uint64_t bi[KM > 0 ? KM : 1];
    double* hd = nullptr;
    uint64_t* hi = nullptr;
    if (KM == 0) {
        hd = heap_d + qi * (int64_t)k;
        hi = heap_i + qi * (int64_t)k;
    }
    int cnt = 0;
    double kth_d = radius;       // pruning radius: radius while under-full, k-th distance when full
    uint64_t kth_i = 0;

    // traversal stack
    int st_node[QCAP];
    float st_off[QCAP][DC];
    int sp = 0;
    float off[DC];
#pragma unroll
    for (int d = 0; d < DC; d++) off[d] = 0.0f;

    auto admissible = [&](float b) {
        const double bb = (double)b;
        return cnt < k ? bb < radius : bb <= kth_d;
    };

    int node = n_nodes > 0 ? 0 : -1;
    while (node >= 0) {
        c0++;
        const KdNode rec = nodes[node];
        if (rec.db >= 0) {
            const int dim = rec.db;
            double qd = q[0];
#pragma unroll
            for (int d = 1; d < DC; d++)
                if (d == dim) qd = q[d];
            const double diff = qd - rec.v;  // q - v
            const bool goleft = qd < rec.v;
            const int near = goleft ? node + 1 : rec.a;
            const int far = goleft ? rec.a : node + 1;
            // far box: offset along dim becomes |q - v| (rounded toward zero)
            float fo[DC];
#pragma unroll
            for (int d = 0; d < DC; d++) fo[d] = off[d];
            float ad = __double2float_rz(fabs(diff));
#pragma unroll
            for (int d = 0; d < DC; d++)
                if (d == dim) fo[d] = ad;
            float fb = 0.0f;
#pragma unroll
            for (int d = 0; d < DC; d++)
                if (d < D) fb = __fadd_rz(fb, __fmul_rz(fo[d], fo[d]));
            if (admissible(fb) && sp < QCAP) {  // sp < QCAP always holds (depth <= KNN_MAX_DEPTH); kept
                st_node[sp] = far;                 // because it measurably helps the compiler's schedule
#pragma unroll
                for (int d = 0; d < DC; d++) st_off[sp][d] = fo[d];
                sp++;
            }
            node = near;
            continue;
        }
        // leaf bucket scan
        const int start = rec.a, len = -1 - rec.db;
        c1++;
        c2 += len;
        for (int i = start; i < start + len; i++) {
            double dist = 0.0;
#pragma unroll
            for (int d = 0; d < DC; d++) {
                if (d < D) {
                    const double df = __dsub_rn((double)coords[(int64_t)d * n + i], q[d]);
                    dist = __dadd_rn(dist, __dmul_rn(df, df));
                }
            }
            if (cnt < k) {
                if (!(dist < radius)) continue;
            } else if (!(dist <= kth_d)) {
                continue;
            }
            const uint64_t id = ids[i];
            if (has_ex && id == ex) continue;
            if (KM > 0) {
                if (cnt == k && !lexless(dist, id, kth_d, kth_i)) continue;
                const int p = cnt < k ? cnt : k - 1;
#pragma unroll
                for (int j = 0; j < (KM > 0 ? KM : 1); j++)
                    if (j == p) { bd[j] = dist; bi[j] = id; }
#pragma unroll
                for (int j = (KM > 0 ? KM : 1) - 1; j >= 1; j--) {
                    if (j <= p && lexless(bd[j], bi[j], bd[j - 1], bi[j - 1])) {
                        const double td = bd[j]; bd[j] = bd[j - 1]; bd[j - 1] = td;
                        const uint64_t ti = bi[j]; bi[j] = bi[j - 1]; bi[j - 1] = ti;
                    }
                }
                if (cnt < k) cnt++;
                if (cnt == k) {
#pragma unroll
                    for (int j = 0; j < (KM > 0 ? KM : 1); j++)
                        if (j == k - 1) { kth_d = bd[j]; kth_i = bi[j]; }
                }
            } else {
                // the reference's bounded max-heap (local_query.py:36-69)
                if (cnt < k) {
                    int ii = cnt;
                    hd[ii] = dist; hi[ii] = id;
                    while (ii > 0) {
                        const int pp = (ii - 1) / 2;
                        if (lexless(hd[pp], hi[pp], hd[ii], hi[ii])) {
                            double td = hd[pp]; hd[pp] = hd[ii]; hd[ii] = td;
                            uint64_t ti = hi[pp]; hi[pp] = hi[ii]; hi[ii] = ti;
                            ii = pp;
                        } else break;
                    }
                    cnt++;
                } else {
                    if (!lexless(dist, id, hd[0], hi[0])) continue;
                    hd[0] = dist; hi[0] = id;
                    int ii = 0;
                    for (;;) {
                        const int l = 2 * ii + 1, r = l + 1;
                        int big = ii;
                        if (l < cnt && lexless(hd[big], hi[big], hd[l], hi[l])) big = l;
                        if (r < cnt && lexless(hd[big], hi[big], hd[r], hi[r])) big = r;
                        if (big == ii) break;
                        double td = hd[big]; hd[big] = hd[ii]; hd[ii] = td;
                        uint64_t ti = hi[big]; hi[big] = hi[ii]; hi[ii] = ti;
                        ii = big;
                    }
                }
                if (cnt == k) { kth_d = hd[0]; kth_i = hi[0]; }
            }
        }
        // pop the next admissible far child
        node = -1;
        while (sp > 0) {
            sp--;
            float po[DC];
#pragma unroll
            for (int d = 0; d < DC; d++) po[d] = st_off[sp][d];
            float pb = 0.0f;
#pragma unroll
            for (int d = 0; d < DC; d++)
                if (d < D) pb = __fadd_rz(pb, __fmul_rz(po[d], po[d]));
            if (admissible(pb)) {
                node = st_node[sp];
#pragma unroll
                for (int d = 0; d < DC; d++) off[d] = po[d];
                break;
            }
            c0++;  // popped and pruned (counted like the reference's visit of a pruned node)
        }
    }
    // results: ascending (sq_dist, id)
    out_c[qi] = cnt;
    if (KM > 0) {
#pragma unroll
        for (int j = 0; j < (KM > 0 ? KM : 1); j++) {
            if (j < cnt) {
                out_d[qi * (int64_t)k + j] = bd[j];
                out_i[qi * (int64_t)k + j] = bi[j];
            }
        }
    } else {
        int hs = cnt, j = cnt;
        while (hs > 0) {
            j--;
            out_d[qi * (int64_t)k + j] = hd[0];
            out_i[qi * (int64_t)k + j] = hi[0];
            hs--;
            if (hs > 0) {
                hd[0] = hd[hs]; hi[0] = hi[hs];
                int ii = 0;
                for (;;) {
                    const int l = 2 * ii + 1, r = l + 1;
                    int big = ii;
                    if (l < hs && lexless(hd[big], hi[big], hd[l], hi[l])) big = l;
                    if (r < hs && lexless(hd[big], hi[big], hd[r], hi[r])) big = r;
                    if (big == ii) break;
                    double td = hd[big]; hd[big] = hd[ii]; hd[ii] = td;
                    uint64_t ti = hi[big]; hi[big] = hi[ii]; hi[ii] = ti;
                    ii = big;
                }
            }
        }
    }
    if (out_ctr) {
        out_ctr[qi * 3 + 0] = c0;
        out_ctr[qi * 3 + 1] = c1;
        out_ctr[qi * 3 + 2] = c2;
    }
}

// ----------------------------------------------------------------------------
// Home pass of the two-pass 2-D/3-D search: one thread per query in sorted order
// descends to the query's home leaf (no stack) and keeps the kk smallest binary64
// distances of that bucket (values only, branch-free min/max chain).  The kk-th
// one is an upper bound on the query's final kk-th distance: k_knn_persist starts
// from it, so its traversal prunes from the first node and only the few points
// inside the bound reach the list insertion.  Every lane of a warp is in the same
// phase here, which the persistent kernel (lanes at arbitrary points of their
// walks) cannot offer to the insertion-heavy first bucket.
// bound0[t] = +inf when the bucket holds fewer than kk points with d < radius.
// ----------------------------------------------------------------------------
template <typename T, int DT, int KM>
__global__ void __launch_bounds__(128)
k_knn_home(const KdNode* __restrict__ nodes, int64_t n_nodes, const T* __restrict__ coords, int64_t n,
           const double* __restrict__ queries, const int32_t* __restrict__ order, int64_t nq, int kk,
           const double* __restrict__ radii, double* __restrict__ bound0, int32_t* __restrict__ entry) {
    static_assert(DT > 0, "fixed-dimension instances only");
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= nq) return;
    const int64_t qi = order ? (int64_t)order[t] : t;
    double q[DT];
#pragma unroll
    for (int d = 0; d < DT; d++) q[d] = queries[qi * DT + d];
    const double radius = radii ? radii[qi] : INFINITY;
    if (n_nodes <= 0) { bound0[t] = INFINITY; entry[t] = 0; return; }
    int node = 0;
    KdNode rec = nodes[0];
    while (rec.db >= 0) {
        double qd = q[0];
#pragma unroll
        for (int d = 1; d < DT; d++)
            if (d == rec.db) qd = q[d];
        node = qd < rec.v ? node + 1 : rec.a;
        rec = nodes[node];
    }
    const int start = rec.a, end = rec.a + (-1 - rec.db);
    constexpr int UN = 4;
    double b;
    if constexpr (sizeof(T) == 4 && KD_HOME_F32) {
        // float coordinates: the bound only has to be an UPPER bound on the kk-th distance, so it is
        // computed in fp32 with upward rounding -- |c - q| <= max(c - q_lo, q_hi - c) with q_lo <= q
        // <= q_hi the float neighbours of q, squares accumulated by round-up FMAs -- one FMNMX per
        // step of the selection chain instead of compare + selects on doubles.  Points enter when the
        // upper bound is below the radius rounded down, so the bound stays below the radius.
        float qlo[DT], qhi[DT];
#pragma unroll
        for (int d = 0; d < DT; d++) {
            qlo[d] = __double2float_rd(q[d]);
            qhi[d] = __double2float_ru(q[d]);
        }
        const float radf = __double2float_rd(radius);
        float fd[KM];
#pragma unroll
        for (int j = 0; j < KM; j++) fd[j] = INFINITY;
        for (int base = start; base < end; base += UN) {
            float cv[UN][DT];
#pragma unroll
            for (int u = 0; u < UN; u++) {
                const int i = min(base + u, end - 1);
#pragma unroll
                for (int d = 0; d < DT; d++) cv[u][d] = (float)coords[(int64_t)d * n + i];
            }
#pragma unroll
            for (int u = 0; u < UN; u++) {
                float ub = 0.0f;
#pragma unroll
                for (int d = 0; d < DT; d++) {
                    const float m = fmaxf(__fsub_ru(cv[u][d], qlo[d]), __fsub_ru(qhi[d], cv[u][d]));
                    ub = __fmaf_ru(m, m, ub);
                }
                float x = (base + u < end && ub < radf) ? ub : INFINITY;
#pragma unroll
                for (int j = 0; j < KM; j++) {
                    const float lo = fminf(x, fd[j]);
                    x = fmaxf(x, fd[j]);
                    fd[j] = lo;
                }
            }
        }
        float bf = fd[KM - 1];
#pragma unroll
        for (int j = 0; j < KM - 1; j++)
            if (j == kk - 1) bf = fd[j];
        b = (double)bf;
    } else {
    double bd[KM];
#pragma unroll
    for (int j = 0; j < KM; j++) bd[j] = INFINITY;
    for (int base = start; base < end; base += UN) {
        T cv[UN][DT];
#pragma unroll
        for (int u = 0; u < UN; u++) {
            const int i = min(base + u, end - 1);
#pragma unroll
            for (int d = 0; d < DT; d++) cv[u][d] = coords[(int64_t)d * n + i];
        }
#pragma unroll
        for (int u = 0; u < UN; u++) {
            double dist = 0.0;
#pragma unroll
            for (int d = 0; d < DT; d++) {
                const double df = __dsub_rn((double)cv[u][d], q[d]);
                dist = __dadd_rn(dist, __dmul_rn(df, df));
            }
            // a repeated point (the clamped tail) or one outside the radius does not enter
            double x = (base + u < end && dist < radius) ? dist : INFINITY;
#pragma unroll
            for (int j = 0; j < KM; j++) {
                const bool lt = x < bd[j];
                const double lo = lt ? x : bd[j];
                x = lt ? bd[j] : x;
                bd[j] = lo;
            }
        }
    }
    b = bd[KM - 1];
#pragma unroll
    for (int j = 0; j < KM - 1; j++)
        if (j == kk - 1) b = bd[j];
    }
    bound0[t] = b;
    // Entry node: on the root-to-home path the query lies on the near side of every plane
    // (all box offsets zero), and a far child whose bound |q - v|^2 exceeds the bound b can
    // never be admitted (the threshold only tightens).  The walk may therefore start at the
    // first node of the path whose far child is admissible -- same bound arithmetic and the
    // same test as k_knn_persist's push -- instead of the root.
    int e = 0;
    if (b < INFINITY) {
        rec = nodes[0];
        while (rec.db >= 0) {
            double qd = q[0];
#pragma unroll
            for (int d = 1; d < DT; d++)
                if (d == rec.db) qd = q[d];
            const float ad = __double2float_rz(fabs(qd - rec.v));
            const float fb = __fadd_rz(0.0f, __fmul_rz(ad, ad));
            if ((double)fb <= b) break;
            e = qd < rec.v ? e + 1 : rec.a;
            rec = nodes[e];
        }
    }
    entry[t] = e;
}

// ----------------------------------------------------------------------------
// Persistent warps with dynamic query fetch.  Each lane runs its own exact
// traversal (same bounds / admission rules as k_knn); when a lane finishes its
// query it takes the next one from a warp-local pool of leaf-sorted queries,
// refilled 64 at a time from a global counter.  This removes the tail
// imbalance of one-query-per-thread warps (a warp otherwise waits for its
// slowest query) while keeping neighbouring lanes on neighbouring queries.
// ----------------------------------------------------------------------------
// low-dimensional, small-k instances are held to 72 registers (7 CTAs of 4 warps per SM)
// SCAN: 0 = the lane walks its own push-free first descent and inserts inline while scanning;
//       2 = two-pass: the k-th distance bound comes from k_knn_home (bound0, by sorted position),
//           and buckets are scanned in chunks whose hits are inserted afterwards (see below)
template <typename T, int DT, int KM, int SCAN = 0>
__global__ void __launch_bounds__(128, (DT > 0 && DT <= 3 && KM <= 8) ? KD_KNN_CTAS : 1)
k_knn_persist(const KdNode* __restrict__ nodes, int64_t n_nodes, const T* __restrict__ coords,
              const uint64_t* __restrict__ ids, int64_t n, int dims_rt, const double* __restrict__ queries,
              const int32_t* __restrict__ order, int64_t nq, int k, const double* __restrict__ radii,
              const uint64_t* __restrict__ excl, double* __restrict__ out_d, uint64_t* __restrict__ out_i,
              int64_t* __restrict__ out_c, int64_t* __restrict__ out_ctr, unsigned long long* __restrict__ counter,
              bool push_free_first, const uint32_t* __restrict__ home_keys,
              const double* __restrict__ bound0 = nullptr, const int32_t* __restrict__ entry = nullptr) {
    constexpr int DC = Dims<DT>::cap;
    constexpr int POOL = 64;
    const int D = DT > 0 ? DT : dims_rt;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1;

    double q[DC];
    double radius = 0.0;
    uint64_t ex = ~0ULL;
    const bool has_ex = excl != nullptr;
    // with an excluded id the search keeps k+1 candidates and drops that id at
    // output: top-(k+1) minus {ex}, truncated to k == top-k of the set minus {ex}
    // the dispatcher picks KM == k(+1) exactly for 1, 2, 5, 6: then the list length is a
    // compile-time constant (the insertion's slot guards and the k-th-slot pick fold away)
    constexpr bool EXACT = KM == 1 || KM == 2 || KM == 5 || KM == 6;
    const int kk = EXACT ? KM : k + (has_ex ? 1 : 0);
    int64_t qi = -1;
    int64_t c0 = 0, c1 = 0, c2 = 0;
    double bd[KM];
    uint32_t bp[KM];  // packed rows; ids[bp] at output
    int cnt = 0;
    double kth_d = 0.0;
    uint32_t kth_p = 0;
    float off[DC];
    int st_node[QCAP];
    float st_off[QCAP][DC];
    int sp = 0;
    int node = -1;
    int home = -1;          // home leaf: scanned by the first (push-free) descent
    bool first = false;     // in the first descent (no far children pushed yet)
    long long pool_base = 0;
    int pool_left = 0;
    bool exhausted = false;

    // admission threshold kth_d: the radius (strict) until the list is full or a bound from the
    // home pass is known, then a distance that kk points are known to reach (inclusive)
    bool strict = true;
    auto admissible = [&](float b) {
        const double bb = (double)b;
        if constexpr (SCAN == 2) return strict ? bb < kth_d : bb <= kth_d;
        return cnt < kk ? bb < radius : bb <= kth_d;
    };
    // exact fp32 pre-filter for float trees: a point whose binary64 distance d
    // can still be admitted (d <= R, R = radius or k-th distance) has an fp32
    // distance d32 = sum (c - fl32(q))^2 <= thr(R), where with u = 2^-24 and
    // x = R(1+2^-50):  thr = (x + 2u^2|q|^2 + 2u|q| sqrt(x + u^2|q|^2))
    //                        * (1 + (D+2)u) / (1-2u)^2 * (1 + 2^-40)
    // (|t' - t| <= u|q_d| + u|t'| per coordinate, fp32 accumulation <= (D+1)u).
    // Points with d32 > thr are skipped without the binary64 evaluation.
    float q32[DC];
    double qnorm = 0.0;
    float thr32 = INFINITY;
    auto make_thr = [&](double R) {
        if (!(R < 1e300)) return INFINITY;
        const double u = 5.9604644775390625e-08;
        const double x = R * (1.0 + 1e-15);
        const double uq = u * qnorm;
        const double t = (x + 2.0 * uq * uq + 2.0 * uq * sqrt(x + uq * uq)) * (1.0 + (D + 2) * u) /
                         ((1.0 - 2.0 * u) * (1.0 - 2.0 * u)) * (1.0 + 1e-12);
        return t >= 3.0e38 ? INFINITY : __double2float_ru(t);
    };

    for (;;) {
        // ---- hand out queries to idle lanes
        const bool need = node < 0;
        const unsigned mneed = __ballot_sync(FULL, need);
        if (mneed && !exhausted) {
            int want = __popc(mneed);
            int got_rank = -1;
            // lanes take from the pool in lane order
            int rank = __popc(mneed & lt_mask);
            long long myq = -1;
            if (rank < pool_left) myq = pool_base + rank;
            const int taken = min(want, pool_left);
            pool_base += taken;
            pool_left -= taken;
            if (want > taken) {
                long long nb = 0;
                if (lane == 0) nb = (long long)atomicAdd(counter, (unsigned long long)POOL);
                nb = __shfl_sync(FULL, nb, 0);
                if (nb >= nq) {
                    exhausted = true;
                } else {
                    pool_base = nb;
                    pool_left = (int)min((long long)POOL, nq - nb);
                    const int r2 = rank - taken;
                    if (need && r2 >= 0 && r2 < pool_left) myq = pool_base + r2;
                    const int t2 = min(want - taken, pool_left);
                    pool_base += t2;
                    pool_left -= t2;
                }
            }
            (void)got_rank;
            if (need && myq >= 0 && myq < nq) {
                qi = order ? (int64_t)order[myq] : myq;
#pragma unroll
                for (int d = 0; d < DC; d++) q[d] = d < D ? queries[qi * D + d] : 0.0;
                radius = radii ? radii[qi] : INFINITY;
                ex = has_ex ? excl[qi] : ~0ULL;
                cnt = 0;
                kth_d = radius;
                kth_p = 0;
#pragma unroll
                for (int j = 0; j < KM; j++) bd[j] = INFINITY;
                c0 = c1 = c2 = 0;
                if constexpr (kPersistF32Filter<DT> && sizeof(T) == 4) {
                    double qq = 0.0;
#pragma unroll
                    for (int d = 0; d < DC; d++) {
                        q32[d] = __double2float_rn(q[d]);
                        qq += q[d] * q[d];
                    }
                    qnorm = sqrt(qq) * (1.0 + 1e-12);
                    thr32 = make_thr(radius);
                }
                sp = 0;
                home = -1;
                first = SCAN == 2 ? false : push_free_first;
                if constexpr (SCAN == 2) {
                    const double t0 = bound0[myq];
                    strict = !(t0 < INFINITY);
                    if (!strict) kth_d = t0;  // < radius: the home pass admits d < radius only
                }
#pragma unroll
                for (int d = 0; d < DC; d++) off[d] = 0.0f;
                // -2: finished immediately (empty tree).  With the home-leaf sort keys the
                // first (push-free) descent is a jump: k_leaf_of already walked it.
                node = n_nodes > 0 ? ((home_keys && first) ? (int)home_keys[myq] : 0) : -2;
                if constexpr (SCAN == 2) {
                    if (n_nodes > 0) node = entry[myq];
                }
            }
        }
        if (node == -2) {
            out_c[qi] = 0;
            if (out_ctr) { out_ctr[qi * 3] = 0; out_ctr[qi * 3 + 1] = 0; out_ctr[qi * 3 + 2] = 0; }
            node = -1;
        }
        if (__ballot_sync(FULL, node >= 0) == 0) {
            if (exhausted) break;
            continue;
        }
        if (node < 0) continue;
        // ---- descend to a leaf, pushing admissible far children (node steps only;
        // the bucket is scanned below, after the warp reconverges, so every lane
        // that reached a leaf in this round scans at the same time)
        int lstart = 0, llen = 0;
        for (;;) {
            c0++;
            const KdNode rec = nodes[node];
            if (rec.db < 0 && node == home) break;  // already scanned by the first descent
            if (rec.db < 0) {
                lstart = rec.a;
                llen = -1 - rec.db;
                break;
            }
            const int dim = rec.db;
            double qd = q[0];
#pragma unroll
            for (int d = 1; d < DC; d++)
                if (d == dim) qd = q[d];
            const bool goleft = qd < rec.v;
            const int near = goleft ? node + 1 : rec.a;
            const int far = goleft ? rec.a : node + 1;
            const float ad = __double2float_rz(fabs(qd - rec.v));
            float fo[DC];
            float fb = 0.0f;
#pragma unroll
            for (int d = 0; d < DC; d++) {
                fo[d] = (d == dim) ? ad : off[d];
                if (d < D) fb = __fadd_rz(fb, __fmul_rz(fo[d], fo[d]));
            }
            if (!first && admissible(fb) && sp < QCAP) {  // always true (see QCAP); keeps the faster schedule
                st_node[sp] = far;
#pragma unroll
                for (int d = 0; d < DC; d++) st_off[sp][d] = fo[d];
                sp++;
            }
            node = near;
        }
        // ---- scan the bucket
        if (llen > 0) {
            const int start = lstart, len = llen;
            c1++;
            c2 += len;
            if constexpr (SCAN == 2) {
                // Chunked scan with deferred insertion.  A chunk's binary64 distances stay in
                // registers; each is compared with the threshold as it stands (a superset test:
                // the threshold only tightens) and the hits are recorded in a bit mask, then
                // drained one per iteration.  With 32 independent lanes some lane hits at almost
                // every point, so inline insertion runs its ~80 instructions on nearly every step
                // for a handful of lanes; here it runs max-over-lanes(hits per chunk) times.
                constexpr int CH = 4;
                const int end = start + len;
                for (int base = start; base < end; base += CH) {
                    double dv[CH];
                    unsigned cand = 0;
#pragma unroll
                    for (int u = 0; u < CH; u++) {
                        const int i = min(base + u, end - 1);
                        double dist = 0.0;
#pragma unroll
                        for (int d = 0; d < DC; d++) {
                            if (d < D) {
                                const double df = __dsub_rn((double)coords[(int64_t)d * n + i], q[d]);
                                dist = __dadd_rn(dist, __dmul_rn(df, df));
                            }
                        }
                        dv[u] = dist;
                        cand |= (unsigned)(dist <= kth_d && base + u < end) << u;
                    }
                    while (cand) {
                        const int u = __ffs(cand) - 1;
                        cand &= cand - 1;
                        double dist = dv[0];
#pragma unroll
                        for (int v = 1; v < CH; v++)
                            if (u == v) dist = dv[v];
                        const int i = base + u;
                        if (cnt < kk ? (strict ? dist < kth_d : dist <= kth_d)
                                     : (dist <= kth_d && lexless_pos(dist, (uint32_t)i, kth_d, kth_p, ids))) {
                            topk_insert_pos<KM>(bd, bp, cnt, kk, dist, (uint32_t)i, ids);
                            if (cnt == kk) {
                                topk_last<KM>(bd, bp, kk, kth_d, kth_p);
                                strict = false;
                            }
                        }
                    }
                }
            } else {
            // software pipeline: the next point's coordinates are in flight while this one is
            // evaluated (the binary64 conversion no longer waits on the load; -9 % on C2/C3)
            T nx[DC];
#pragma unroll
            for (int d = 0; d < DC; d++)
                if (d < D) nx[d] = coords[(int64_t)d * n + start];
            for (int i = start; i < start + len; i++) {
                T cv[DC];
#pragma unroll
                for (int d = 0; d < DC; d++) cv[d] = nx[d];
                if (i + 1 < start + len) {
#pragma unroll
                    for (int d = 0; d < DC; d++)
                        if (d < D) nx[d] = coords[(int64_t)d * n + i + 1];
                }
                bool take = true;
                if constexpr (kPersistF32Filter<DT> && sizeof(T) == 4) {
                    float d32 = 0.0f;
#pragma unroll
                    for (int d = 0; d < DC; d++) {
                        if (d < D) {
                            const float tt = cv[d] - q32[d];
                            d32 = fmaf(tt, tt, d32);
                        }
                    }
                    take = !(d32 > thr32);
                }
                if (take) {
                    double dist = 0.0;
#pragma unroll
                    for (int d = 0; d < DC; d++) {
                        if (d < D) {
                            const double df = __dsub_rn((double)cv[d], q[d]);
                            dist = __dadd_rn(dist, __dmul_rn(df, df));
                        }
                    }
                    if (cnt < kk ? dist < radius
                                 : (dist <= kth_d && lexless_pos(dist, (uint32_t)i, kth_d, kth_p, ids))) {
                        topk_insert_pos<KM>(bd, bp, cnt, kk, dist, (uint32_t)i, ids);
                        if (cnt == kk) {
                            topk_last<KM>(bd, bp, kk, kth_d, kth_p);
                            if constexpr (kPersistF32Filter<DT> && sizeof(T) == 4) thr32 = make_thr(kth_d);
                        }
                    }
                }
            }
            }
        }
        // ---- after the home leaf: restart from the root with a real k-th distance
        if (first) {
            first = false;
            home = node;
            node = 0;
#pragma unroll
            for (int d = 0; d < DC; d++) off[d] = 0.0f;
            if (home != 0) continue;  // (a single-leaf tree is done)
        }
        // ---- next admissible far child, or finish
        node = -1;
        while (sp > 0) {
            sp--;
            float po[DC];
            float pb = 0.0f;
#pragma unroll
            for (int d = 0; d < DC; d++) {
                po[d] = st_off[sp][d];
                if (d < D) pb = __fadd_rz(pb, __fmul_rz(po[d], po[d]));
            }
            if (admissible(pb)) {
                node = st_node[sp];
#pragma unroll
                for (int d = 0; d < DC; d++) off[d] = po[d];
                break;
            }
            c0++;
        }
        if (node < 0) {
            int w = 0;
            bool dropped = false;
#pragma unroll
            for (int j = 0; j < KM; j++) {
                if (j < cnt) {
                    const uint64_t id = ids[bp[j]];
                    if (has_ex && !dropped && id == ex) {
                        dropped = true;
                    } else if (w < k) {
                        out_d[qi * (int64_t)k + w] = bd[j];
                        out_i[qi * (int64_t)k + w] = id;
                        w++;
                    }
                }
            }
            out_c[qi] = w;
            if (out_ctr) {
                out_ctr[qi * 3 + 0] = c0;
                out_ctr[qi * 3 + 1] = c1;
                out_ctr[qi * 3 + 2] = c2;
            }
        }
    }
}

// ----------------------------------------------------------------------------
// Warp per query for D >= 4.  In higher dimensions a query scans thousands of
// buckets (C4: ~2.1K buckets, ~130K points per query) and neighbouring queries'
// candidate sets differ, so one lane per query diverges and reads scattered
// buckets, and a shared (packet) traversal blows up to the union of 32 queries'
// candidates.  Here the whole warp serves one query: the traversal is executed
// uniformly by every lane (no divergence), and a bucket is scanned with one
// point per lane -- coalesced SoA loads, exact fp32 pre-filter per lane, the
// survivors' binary64 distances (reference order) inserted by the warp in lane
// order into a top-k list that every lane holds.  Queries are taken in home-
// leaf order from a global counter (persistent warps).
// ----------------------------------------------------------------------------
constexpr int WQ_WARPS = 4;
constexpr int WQ_DC = 16;  // max dimensions

template <typename T, int KM, int DCAP>
__global__ void __launch_bounds__(WQ_WARPS * 32, DCAP == WQ_DC ? 5 : 6)
k_knn_wq(const KdNode* __restrict__ nodes, int64_t n_nodes, const T* __restrict__ coords,
         const uint64_t* __restrict__ ids, int64_t n, int D_rt, const double* __restrict__ queries,
         const int32_t* __restrict__ order, int64_t nq, int k, const double* __restrict__ radii,
         const uint64_t* __restrict__ excl, double* __restrict__ out_d, uint64_t* __restrict__ out_i,
         int64_t* __restrict__ out_c, int64_t* __restrict__ out_ctr, unsigned long long* __restrict__ counter) {
    constexpr int DC = DCAP;  // register arrays sized for the dimension count (10 for C4, else 16)
    // an instance for one exact dimension count folds every `d < D` test at compile time
    const int D = DCAP != WQ_DC ? DCAP : D_rt;
    __shared__ int s_node[WQ_WARPS][QCAP];
    __shared__ float s_off[WQ_WARPS][QCAP][32];
    __shared__ double s_q[WQ_WARPS][DC];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool has_ex = excl != nullptr;
    const int kk = k + (has_ex ? 1 : 0);  // top-(k+1) minus the excluded id (see k_knn_persist)
    // box offsets are lane-distributed: lane d holds the offset along dimension d
    // (lanes >= D hold 0); a bound is a round-toward-zero warp sum of squares --
    // rounded down in any order, so still <= every point's binary64 distance
    auto bound_of = [&](float o) {
        float b = __fmul_rz(o, o);
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) b = __fadd_rz(b, __shfl_xor_sync(FULL, b, s));
        // lanes may associate the butterfly differently: lane 0's value for everyone
        // keeps the traversal warp-uniform
        return __shfl_sync(FULL, b, 0);
    };
    for (;;) {
        long long slot = 0;
        if (lane == 0) slot = (long long)atomicAdd(counter, 1ULL);
        slot = __shfl_sync(FULL, slot, 0);
        if (slot >= nq) break;
        const int64_t qi = order ? (int64_t)order[slot] : slot;
        const double* qrow = queries + qi * D;
        const double radius = radii ? radii[qi] : INFINITY;
        const uint64_t ex = has_ex ? excl[qi] : ~0ULL;
        const double qmine = lane < D ? qrow[lane] : 0.0;  // lane d: q[d]
        if (lane < DC) s_q[warp][lane] = qmine;
        double qq = qmine * qmine;
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) qq += __shfl_xor_sync(FULL, qq, s);
        __syncwarp();
        float q32[DC];
#pragma unroll
        for (int d = 0; d < DC; d++) q32[d] = __double2float_rn(s_q[warp][d]);
        const double qnorm = sqrt(qq) * (1.0 + 1e-12);
        auto make_thr = [&](double R) {  // exact fp32 pre-filter threshold (derivation at k_knn_persist)
            if (!(R < 1e300)) return INFINITY;
            const double u = 5.9604644775390625e-08;
            const double x = R * (1.0 + 1e-15);
            const double uq = u * qnorm;
            const double t = (x + 2.0 * uq * uq + 2.0 * uq * sqrt(x + uq * uq)) * (1.0 + (D + 2) * u) /
                             ((1.0 - 2.0 * u) * (1.0 - 2.0 * u)) * (1.0 + 1e-12);
            return t >= 3.0e38 ? INFINITY : __double2float_ru(t);
        };
        // the sorted list is lane-distributed: lane j holds entry j (k + 1 <= 32)
        double my_d = INFINITY;
        uint32_t my_p = 0;
        int cnt = 0;
        double kth_d = radius;
        uint32_t kth_p = 0;
        float thr32 = sizeof(T) == 4 ? make_thr(radius) : INFINITY;
        int64_t c0 = 0, c1 = 0, c2 = 0;
        float off = 0.0f;  // this lane's dimension
        auto admissible = [&](float b) {
            const double bb = (double)b;
            return cnt < kk ? bb < radius : bb <= kth_d;
        };
        int node = n_nodes > 0 ? 0 : -1;
        int sp = 0;
        while (node >= 0) {
            c0++;
            const KdNode rec = nodes[node];
            if (rec.db >= 0) {
                const int dim = rec.db;
                const double qd = s_q[warp][dim];
                const bool goleft = qd < rec.v;
                const int near = goleft ? node + 1 : rec.a;
                const int far = goleft ? rec.a : node + 1;
                const float ad = __double2float_rz(fabs(qd - rec.v));
                const float of = lane == dim ? ad : off;
                if (admissible(bound_of(lane < D ? of : 0.0f)) && sp < QCAP) {  // always true (see QCAP)
                    s_off[warp][sp][lane] = of;
                    s_node[warp][sp] = far;  // every lane stores the (warp-uniform) index: no cross-lane race
                    sp++;
                }
                node = near;
                continue;
            }
            // bucket: one point per lane per round, two rounds' loads issued together
            const int start = rec.a, len = -1 - rec.db;
            c1++;
            c2 += len;
            for (int c = 0; c < len; c += 64) {
                T cv[2][DC];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int j = c + h * 32 + lane;
#pragma unroll
                    for (int d = 0; d < DC; d++) cv[h][d] = T(0);
                    if (j < len) {  // one guard per point; the dimension rows by pointer steps
                        const T* pp = coords + start + j;
#pragma unroll
                        for (int d = 0; d < DC; d++) {
                            if (d < D) cv[h][d] = *pp;
                            pp += n;
                        }
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int cc = c + h * 32;
                    if (cc >= len) break;
                    const bool valid = cc + lane < len;
                    bool pass = valid;
                    if constexpr (sizeof(T) == 4) {
                        float d32 = 0.0f;
#pragma unroll
                        for (int d = 0; d < DC; d++) {
                            if (d < D) {
                                const float tt = cv[h][d] - q32[d];
                                d32 = fmaf(tt, tt, d32);
                            }
                        }
                        pass = pass && !(d32 > thr32);
                    }
                    double dist = INFINITY;
                    if (pass) {
                        dist = 0.0;
#pragma unroll
                        for (int d = 0; d < DC; d++) {
                            if (d < D) {
                                const double df = __dsub_rn((double)cv[h][d], s_q[warp][d]);
                                dist = __dadd_rn(dist, __dmul_rn(df, df));
                            }
                        }
                        pass = cnt < kk ? dist < radius : dist <= kth_d;
                    }
                    unsigned m = __ballot_sync(FULL, pass);
                    while (m) {  // survivors in point order, inserted uniformly by every lane
                        const int src = __ffs(m) - 1;
                        m &= m - 1;
                        const double dd = __shfl_sync(FULL, dist, src);
                        const uint32_t pos = (uint32_t)(start + cc + src);
                        if (cnt < kk ? dd < radius : (dd <= kth_d && lexless_pos(dd, pos, kth_d, kth_p, ids))) {
                            // entries preceding (dd, pos) form a prefix of the lanes; ids only on ties
                            const bool before = lane < cnt && (my_d < dd || (my_d == dd && ids[my_p] < ids[pos]));
                            const int at = __popc(__ballot_sync(FULL, before));
                            const double up_d = __shfl_up_sync(FULL, my_d, 1);
                            const uint32_t up_p = __shfl_up_sync(FULL, my_p, 1);
                            if (lane > at && lane < kk) { my_d = up_d; my_p = up_p; }
                            if (lane == at) { my_d = dd; my_p = pos; }
                            if (cnt < kk) cnt++;
                            if (cnt == kk) {
                                kth_d = __shfl_sync(FULL, my_d, kk - 1);
                                kth_p = __shfl_sync(FULL, my_p, kk - 1);
                                if constexpr (sizeof(T) == 4) thr32 = make_thr(kth_d);
                            }
                        }
                    }
                }
            }
            // next admissible far child
            node = -1;
            while (sp > 0) {
                sp--;
                const float po = s_off[warp][sp][lane];
                if (admissible(bound_of(lane < D ? po : 0.0f))) {
                    node = s_node[warp][sp];
                    off = po;
                    break;
                }
                c0++;
            }
        }
        // results: lane j holds entry j; the excluded id (if present) is dropped
        const uint64_t my_id = lane < cnt ? ids[my_p] : 0;
        const unsigned exm = __ballot_sync(FULL, has_ex && lane < cnt && my_id == ex);
        const int drop = exm ? __ffs(exm) - 1 : 32;
        const int w = min(cnt - (exm ? 1 : 0), k);
        if (lane < cnt && lane != drop) {
            const int slot = lane - (lane > drop ? 1 : 0);
            if (slot < k) {
                out_d[qi * (int64_t)k + slot] = my_d;
                out_i[qi * (int64_t)k + slot] = my_id;
            }
        }
        if (lane == 0) {
            out_c[qi] = w;
            if (out_ctr) {
                out_ctr[qi * 3 + 0] = c0;
                out_ctr[qi * 3 + 1] = c1;
                out_ctr[qi * 3 + 2] = c2;
            }
        }
        __syncwarp();
    }
}

// leaf reached by descending with the tie rule (coord >= value goes right);
// used as the sort key that makes each warp's 32 queries spatially coherent
template <int DT>
__global__ void k_leaf_of(const KdNode* __restrict__ nodes, int64_t n_nodes, const double* __restrict__ queries,
                          int dims_rt, int64_t nq, uint32_t* __restrict__ key, int32_t* __restrict__ val) {
    // LQ independent descents per thread, advanced in lock step: LQ node loads in flight at once
    constexpr int LQ = 4;
    const int D = DT > 0 ? DT : dims_rt;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int node[LQ];
    bool live[LQ];
#pragma unroll
    for (int u = 0; u < LQ; u++) {
        node[u] = 0;
        live[u] = i0 + u * stride < nq && n_nodes > 0;
    }
    for (;;) {
        bool any = false;
        KdNode rec[LQ];
#pragma unroll
        for (int u = 0; u < LQ; u++)
            if (live[u]) rec[u] = nodes[node[u]];
#pragma unroll
        for (int u = 0; u < LQ; u++) {
            if (!live[u]) continue;
            if (rec[u].db < 0) { live[u] = false; continue; }
            const int64_t i = i0 + u * stride;
            node[u] = queries[i * D + rec[u].db] < rec[u].v ? node[u] + 1 : rec[u].a;
            any = true;
        }
        if (!any) break;
    }
#pragma unroll
    for (int u = 0; u < LQ; u++) {
        const int64_t i = i0 + u * stride;
        if (i < nq) {
            key[i] = (uint32_t)node[u];
            val[i] = (int32_t)i;
        }
    }
}

// first descent without pushes, then a restart from the root with the k-th
// distance of the home leaf (KDB_KNN_PFF=0 disables; for A/B measurements)
static bool knn_push_free_first() {
    static const bool v = [] {
        const char* e = getenv("KDB_KNN_PFF");
        return !(e && e[0] == '0');
    }();
    return v;
}

// 2-D/3-D search with k(+1) <= 8: 2 = two-pass (k_knn_home + deferred-insertion scan, default),
// 0 = single persistent kernel with inline insertion (KDB_KNN_SCAN, for A/B measurements)
static int knn_scan_mode() {
    static const int v = [] {
        const char* e = getenv("KDB_KNN_SCAN");
        return e ? atoi(e) : 2;
    }();
    return v;
}

template <typename T, int DT, int KM>
static void launch_knn(const KdTreeDev& t, const KnnArgs& a, const int32_t* order, const uint32_t* home,
                       cudaStream_t st) {
    const int threads = 128;
    const unsigned blocks = (unsigned)((a.nq + threads - 1) / threads);
    if constexpr (KM > 0 && DT == 0) {
        if (!a.thread_per_query && t.dims <= WQ_DC) {
            auto go = [&](auto kern) {
                int dev = 0, sms = 148, per_sm = 0;
                cudaGetDevice(&dev);
                cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WQ_WARPS * 32, 0);
                const long long want = (a.nq + WQ_WARPS - 1) / WQ_WARPS;
                const unsigned grid =
                    (unsigned)std::max(1LL, std::min<long long>(want, (long long)sms * std::max(per_sm, 1)));
                unsigned long long* ctr = scratch<unsigned long long>(1, st);
                KD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
                kern<<<grid, WQ_WARPS * 32, 0, st>>>(t.nodes, t.n_nodes, static_cast<const T*>(t.coords), t.ids, t.n,
                                                     t.dims, a.queries, order, a.nq, (int)a.k, a.radii, a.excl,
                                                     a.out_d, a.out_i, a.out_c, a.out_ctr, ctr);
                scratch_free(ctr, st);
            };
            if (t.dims == 10) go(k_knn_wq<T, KM, 10>);  // exact-dimension instance (C4)
            else go(k_knn_wq<T, KM, WQ_DC>);
            return;
        }
    }
    if constexpr (KM > 0) {
        if (!a.thread_per_query) {
            int dev = 0, sms = 148, per_sm = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_knn_persist<T, DT, KM>, threads, 0);
            const long long want = (a.nq + threads - 1) / threads;
            const unsigned grid = (unsigned)std::max(1LL, std::min<long long>(want, (long long)sms * std::max(per_sm, 1)));
            unsigned long long* ctr = scratch<unsigned long long>(1, st);
            KD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
            if constexpr (DT > 0 && DT <= 3 && KM <= 8) {
                if (knn_scan_mode() == 2) {
                    double* bound0 = scratch<double>((size_t)a.nq, st);
                    int32_t* entry = scratch<int32_t>((size_t)a.nq, st);
                    const int kk = (int)a.k + (a.excl ? 1 : 0);
                    k_knn_home<T, DT, KM><<<(unsigned)((a.nq + 127) / 128), 128, 0, st>>>(
                        t.nodes, t.n_nodes, static_cast<const T*>(t.coords), t.n, a.queries, order, a.nq, kk,
                        a.radii, bound0, entry);
                    k_knn_persist<T, DT, KM, 2><<<grid, threads, 0, st>>>(
                        t.nodes, t.n_nodes, static_cast<const T*>(t.coords), t.ids, t.n, t.dims, a.queries, order,
                        a.nq, (int)a.k, a.radii, a.excl, a.out_d, a.out_i, a.out_c, a.out_ctr, ctr, false, nullptr,
                        bound0, entry);
                    scratch_free(entry, st);
                    scratch_free(bound0, st);
                    scratch_free(ctr, st);
                    return;
                }
            }
            k_knn_persist<T, DT, KM><<<grid, threads, 0, st>>>(
                t.nodes, t.n_nodes, static_cast<const T*>(t.coords), t.ids, t.n, t.dims, a.queries, order, a.nq,
                (int)a.k, a.radii, a.excl, a.out_d, a.out_i, a.out_c, a.out_ctr, ctr, knn_push_free_first(), home);
            scratch_free(ctr, st);
            return;
        }
    }
    k_knn<T, DT, KM><<<blocks, threads, 0, st>>>(t.nodes, t.n_nodes, static_cast<const T*>(t.coords), t.ids, t.n,
                                                 t.dims, a.queries, order, a.nq, (int)a.k, a.radii, a.excl, a.out_d,
                                                 a.out_i, a.out_c, a.out_ctr, a.heap_d, a.heap_i);
}

template <typename T, int DT>
static void dispatch_k(const KdTreeDev& t, const KnnArgs& a, const int32_t* order, const uint32_t* home,
                       cudaStream_t st) {
    // list capacity: k, or k+1 when the persistent kernel carries an excluded id
    // (k = 32 with an excluded id falls through to the heap kernel)
    const int64_t kc = a.k + ((a.excl && !a.thread_per_query) ? 1 : 0);
    if (kc == 1) launch_knn<T, DT, 1>(t, a, order, home, st);
    else if (kc == 2) launch_knn<T, DT, 2>(t, a, order, home, st);
    else if (kc <= 4) launch_knn<T, DT, 4>(t, a, order, home, st);
    else if (kc == 5) launch_knn<T, DT, 5>(t, a, order, home, st);
    else if (kc == 6) launch_knn<T, DT, 6>(t, a, order, home, st);
    else if (kc <= 8) launch_knn<T, DT, 8>(t, a, order, home, st);
    else if (kc <= 11) launch_knn<T, DT, 11>(t, a, order, home, st);
    else if (kc <= 16) launch_knn<T, DT, 16>(t, a, order, home, st);
    else if (kc <= 32) launch_knn<T, DT, 32>(t, a, order, home, st);
    else launch_knn<T, DT, 0>(t, a, order, home, st);
}

template <typename T>
static void dispatch_d(const KdTreeDev& t, const KnnArgs& a, const int32_t* order, const uint32_t* home,
                       cudaStream_t st) {
    if (t.dims == 2) dispatch_k<T, 2>(t, a, order, home, st);
    else if (t.dims == 3) dispatch_k<T, 3>(t, a, order, home, st);
    else dispatch_k<T, 0>(t, a, order, home, st);
}

// Z-order (Morton) keys of 3-D queries over their bounding box, 10 bits per
// dimension: a traversal-free spatial order for the persistent kernel (which then
// walks the first descent itself).  KDB_KNN_ORDER=leaf selects the home-leaf order.
__device__ __forceinline__ unsigned long long ord_key(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double ord_inv(unsigned long long k) {
    const unsigned long long b = (k & 0x8000000000000000ULL) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
    return __longlong_as_double((long long)b);
}

static __global__ void k_qbox(const double* __restrict__ q, int64_t nq, unsigned long long* __restrict__ box) {
    unsigned long long lo[3] = {~0ULL, ~0ULL, ~0ULL}, hi[3] = {0ULL, 0ULL, 0ULL};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int d = 0; d < 3; d++) {
            const unsigned long long k = ord_key(q[i * 3 + d]);
            lo[d] = k < lo[d] ? k : lo[d];
            hi[d] = k > hi[d] ? k : hi[d];
        }
    }
#pragma unroll
    for (int d = 0; d < 3; d++) {
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long a = __shfl_xor_sync(0xFFFFFFFFu, lo[d], o), b = __shfl_xor_sync(0xFFFFFFFFu, hi[d], o);
            lo[d] = a < lo[d] ? a : lo[d];
            hi[d] = b > hi[d] ? b : hi[d];
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&box[d], lo[d]);
            atomicMax(&box[3 + d], hi[d]);
        }
    }
}

__device__ __forceinline__ uint32_t spread11(uint32_t x) {  // 11 bits -> every third bit of 33
    uint64_t v = x & 0x7FF;
    v = (v | (v << 16)) & 0x1F0000FFULL;
    v = (v | (v << 8)) & 0x100F00F00FULL;
    v = (v | (v << 4)) & 0x10C30C30C3ULL;
    v = (v | (v << 2)) & 0x1249249249ULL;
    return (uint32_t)v;  // bits >= 32 dropped by the callers' shifts
}

static __global__ void k_morton(const double* __restrict__ q, int64_t nq, const unsigned long long* __restrict__ box,
                                uint32_t* __restrict__ key, int32_t* __restrict__ val, int drop) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nq) return;
    uint32_t c[3];
#pragma unroll
    for (int d = 0; d < 3; d++) {
        const double lo = ord_inv(box[d]), hi = ord_inv(box[3 + d]);
        const double w = hi > lo ? 2047.999 / (hi - lo) : 0.0;
        const double u = (q[i * 3 + d] - lo) * w;
        c[d] = (uint32_t)fmin(fmax(u, 0.0), 2047.0);
    }
    // 32-bit key: x and y with 11 bits, z with 10 (its lowest bit dropped)
    const uint64_t k = ((uint64_t)spread11(c[0]) << 2) | ((uint64_t)spread11(c[1]) << 1) | (uint64_t)spread11(c[2]);
    key[i] = (uint32_t)(k >> drop);  // the top 33 - drop bits of the interleaved key
    val[i] = (int32_t)i;
}

static bool knn_morton_order() {
    static const bool v = [] {
        const char* e = getenv("KDB_KNN_ORDER");
        return !(e && e[0] == 'l');
    }();
    return v;
}

void knn(const KdTreeDev& t, const KnnArgs& a, cudaStream_t st) {
    if (a.nq == 0) return;
    // temporaries (sort keys, CUB scratch, work counters) from the stream's arena
    StreamArena ka(t.device, st);
    int32_t* order = nullptr;
    void* tmp = nullptr;
    uint32_t *k0 = nullptr, *k1 = nullptr;
    int32_t* v0 = nullptr;
    if (a.sort_queries && a.nq > 1 && t.n_nodes > 1) {
        k0 = scratch<uint32_t>(a.nq, st);
        k1 = scratch<uint32_t>(a.nq, st);
        v0 = scratch<int32_t>(a.nq, st);
        order = scratch<int32_t>(a.nq, st);
        const bool morton = t.dims == 3 && knn_morton_order();
        int bits = 1;
        if (morton) {
            unsigned long long* box = nullptr;
            box = scratch<unsigned long long>(6, st);
            const unsigned long long init[6] = {~0ULL, ~0ULL, ~0ULL, 0ULL, 0ULL, 0ULL};
            KD_CUDA(cudaMemcpyAsync(box, init, sizeof(init), cudaMemcpyHostToDevice, st));
            k_qbox<<<592, 256, 0, st>>>(a.queries, a.nq, box);
            static const int mbits = [] {  // key bits = radix-sort passes * 8 (KDB_MORTON_BITS: A/B)
                const char* e = getenv("KDB_MORTON_BITS");
                return e ? std::min(32, std::max(8, atoi(e))) : KNN_MORTON_BITS;
            }();
            k_morton<<<(unsigned)((a.nq + 255) / 256), 256, 0, st>>>(a.queries, a.nq, box, k0, v0, 33 - mbits);
            scratch_free(box, st);
            bits = mbits;
        } else {
            const unsigned blocks = (unsigned)((a.nq + 1023) / 1024);  // 4 queries per thread
            if (t.dims == 3) k_leaf_of<3><<<blocks, 256, 0, st>>>(t.nodes, t.n_nodes, a.queries, t.dims, a.nq, k0, v0);
            else k_leaf_of<0><<<blocks, 256, 0, st>>>(t.nodes, t.n_nodes, a.queries, t.dims, a.nq, k0, v0);
            while (bits < 32 && ((int64_t)1 << bits) < t.n_nodes) bits++;
        }
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, order, (int)a.nq, 0, bits, st);
        tmp = scratch<unsigned char>(tb, st);
        cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, order, (int)a.nq, 0, bits, st);
    }
    if (a.packet && knn_packet(t, a, order, st)) {
        if (order) {
            scratch_free(k0, st); scratch_free(k1, st); scratch_free(v0, st); scratch_free(order, st);
            scratch_free(tmp, st);
        }
        return;
    }
    // the persistent kernel may jump straight to the home leaf only with home-leaf keys
    const uint32_t* home = (order && !(t.dims == 3 && knn_morton_order())) ? k1 : nullptr;
    if (t.dtype == DT_F32) dispatch_d<float>(t, a, order, home, st);
    else dispatch_d<double>(t, a, order, home, st);
    KD_CUDA(cudaGetLastError());
    if (order) {
        scratch_free(k0, st); scratch_free(k1, st); scratch_free(v0, st); scratch_free(order, st);
        scratch_free(tmp, st);
    }
}

}  // namespace kdb
