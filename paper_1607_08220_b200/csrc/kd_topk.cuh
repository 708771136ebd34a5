// kd_topk.cuh -- per-query bounded top-k lists shared by the KNN kernels.
//
// Ordering is the brute-force oracle's (pkg/tests/conftest.py:8-18): ascending
// (sq_dist, point_id).  Lists are keyed by (sq_dist, packed row) and ids are
// read only to break exact distance ties, which preserves the (d, id) order.
#pragma once
#include <stdint.h>

#include "kd_common.cuh"

namespace kdb {

__device__ __forceinline__ bool lexless(double d0, uint64_t i0, double d1, uint64_t i1) {
    return d0 < d1 || (d0 == d1 && i0 < i1);
}

// same list keyed by (sq_dist, packed row): ids are only read to break exact
// distance ties (lexicographic (d, id) order is preserved exactly)
__device__ __forceinline__ bool lexless_pos(double d0, uint32_t p0, double d1, uint32_t p1,
                                            const uint64_t* __restrict__ ids) {
    return d0 < d1 || (d0 == d1 && ids[p0] < ids[p1]);
}

// insert into the ascending (d, packed row) list of capacity k <= KM (the caller
// has checked that it enters): one descending pass, each slot keeps, shifts from
// its predecessor, or takes the new entry; ids are read only on exact ties
template <int KM>
__device__ __forceinline__ void topk_insert_pos_tie(double (&bd)[KM], uint32_t (&bp)[KM], int& cnt, int k, double d,
                                                    uint32_t p, const uint64_t* __restrict__ ids) {
    const int last = cnt < k ? cnt : k - 1;
    bool placed = false;
#pragma unroll
    for (int jj = KM - 1; jj >= 0; jj--) {
        if (jj <= last && !placed) {
            const int pj = jj > 0 ? jj - 1 : 0;
            const bool shift = jj > 0 && (d < bd[pj] || (d == bd[pj] && ids[p] < ids[bp[pj]]));
            if (shift) {
                bd[jj] = bd[pj];
                bp[jj] = bp[pj];
            } else {
                bd[jj] = d;
                bp[jj] = p;
                placed = true;
            }
        }
    }
    if (cnt < k) cnt++;
}

// Slots at or beyond the fill count hold +inf (the kernels initialise the list so),
// so without an exact distance tie each slot j either keeps its entry (it is below d),
// takes d (its predecessor is below d, it is not), or takes its predecessor: one
// comparison per slot and selects, no branches.  A tie with a listed distance (rare)
// takes the id-ordered path above.
template <int KM>
__device__ __forceinline__ void topk_insert_pos(double (&bd)[KM], uint32_t (&bp)[KM], int& cnt, int k, double d,
                                                uint32_t p, const uint64_t* __restrict__ ids) {
    bool tie = false;
#pragma unroll
    for (int j = 0; j < KM; j++) tie |= bd[j] == d;
    if (tie) {
        topk_insert_pos_tie<KM>(bd, bp, cnt, k, d, p, ids);
        return;
    }
    bool below[KM];
#pragma unroll
    for (int j = 0; j < KM; j++) below[j] = bd[j] < d;
#pragma unroll
    for (int j = KM - 1; j >= 0; j--) {
        if (j < k && !below[j]) {
            const bool here = j == 0 || below[j > 0 ? j - 1 : 0];
            bd[j] = here ? d : bd[j > 0 ? j - 1 : 0];
            bp[j] = here ? p : bp[j > 0 ? j - 1 : 0];
        }
    }
    if (cnt < k) cnt++;
}

// slot k-1 of the list (a register move when the list is exactly k long)
template <int KM>
__device__ __forceinline__ void topk_last(const double (&bd)[KM], const uint32_t (&bp)[KM], int k, double& kd,
                                          uint32_t& kp) {
    if (k == KM) {
        kd = bd[KM - 1];
        kp = bp[KM - 1];
        return;
    }
#pragma unroll
    for (int j = 0; j < KM; j++)
        if (j == k - 1) { kd = bd[j]; kp = bp[j]; }
}

// exact fp32 pre-filter threshold for float trees (local_query.py:120-124 contract):
// a point whose binary64 distance d can still be admitted (d <= R) has an fp32
// distance d32 = sum (c - fl32(q))^2 (fmaf accumulation) <= thr(R), where with
// u = 2^-24 and x = R(1 + 1e-15):
//     thr = (x + 2u^2|q|^2 + 2u|q| sqrt(x + u^2|q|^2)) (1 + (D+2)u) / (1-2u)^2 (1 + 1e-12)
// (|t' - t| <= u|q_d| + u|t'| per coordinate, fp32 accumulation <= (D+1)u).
// Points with d32 > thr are skipped without the binary64 evaluation.
__device__ __forceinline__ float f32_filter_thr(double R, double qnorm, int D) {
    if (!(R < 1e300)) return INFINITY;
    const double u = 5.9604644775390625e-08;
    const double x = R * (1.0 + 1e-15);
    const double uq = u * qnorm;
    const double t = (x + 2.0 * uq * uq + 2.0 * uq * sqrt(x + uq * uq)) * (1.0 + (D + 2) * u) /
                     ((1.0 - 2.0 * u) * (1.0 - 2.0 * u)) * (1.0 + 1e-12);
    return t >= 3.0e38 ? INFINITY : __double2float_ru(t);
}

}  // namespace kdb
