// kd_packet.cu -- packet KNN for low-dimensional trees (D <= 3): one warp per
// 32 spatially adjacent queries (Morton order), one shared traversal.
//
// Reference: Algorithm 1 of local_query.py:72-172 (per-query DFS with an
// explicit stack, near child first, prune a subtree whose lower bound exceeds
// the current k-th distance, scan leaf buckets, bounded (d, id) heap).  The
// answer set is fixed by the (sq_dist, point_id) order and the strict radius,
// not by the visiting order, so the B200 kernel is free to reorganise the walk:
//
//  * the 32 lanes of a warp hold 32 Morton-adjacent queries and walk ONE
//    stack of subtrees together (warp-uniform control flow: no divergence
//    between traversals);
//  * every subtree carries a tight f32 bounding box of its points (QNode: the
//    parent stores both children's boxes, 64 B per interior node, built once
//    per tree by k_qlinks/k_qboxes).  Each lane's lower bound is the squared
//    box distance evaluated with round-down f32 steps against a rounded-out
//    f32 bracket of its binary64 query, which is provably <= the binary64
//    distance (reference operation order) of every point in the box, so a
//    subtree is skipped only when it cannot hold a neighbour for ANY lane;
//  * a leaf bucket is staged once in shared memory (one point per lane,
//    coalesced SoA loads) and every lane scans it against its own query: an
//    exact fp32 pre-filter, then the binary64 distance in the reference's
//    order (core.py:199-228: ascending dimension, no FMA) for the survivors;
//  * top-k in registers, keyed by (d, packed row), ids read only on ties
//    (kd_topk.cuh); admission and pruning follow the brute-force oracle
//    (strict radius while under-full, replace on (d, id), prune at bound > r').
//
// The stack lives in shared memory, sized from the tree depth (a DFS that
// pushes only far children holds at most one entry per level).
#include <cub/cub.cuh>

#include <algorithm>

#include "kd_common.cuh"
#include "kd_query.cuh"
#include "kd_topk.cuh"
#include "kd_tree.cuh"
#include "kd_warp.cuh"

namespace kdb {

static_assert(sizeof(QNode) == 64, "QNode is one 64-byte record");

// ---------------------------------------------------------------------------
// query-tree construction: child links, then tight boxes bottom-up
// ---------------------------------------------------------------------------
__global__ void k_qlinks(const KdNode* __restrict__ nodes, int64_t nn, QNode* __restrict__ qn,
                         int32_t* __restrict__ parent) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
    if (i == 0) parent[0] = -1;
    const KdNode rec = nodes[i];
    if (rec.db < 0) return;
    const int32_t L = (int32_t)i + 1, R = rec.a;
    parent[L] = (int32_t)i;
    parent[R] = (int32_t)i;
    const KdNode a = nodes[L], b = nodes[R];
    int4 lk;
    lk.x = a.db < 0 ? a.a : L;
    lk.y = a.db < 0 ? -1 - a.db : -1;
    lk.z = b.db < 0 ? b.a : R;
    lk.w = b.db < 0 ? -1 - b.db : -1;
    *reinterpret_cast<int4*>(&qn[i].l) = lk;
}

__device__ __forceinline__ float box_lo(float v) { return v; }
__device__ __forceinline__ float box_hi(float v) { return v; }
__device__ __forceinline__ float box_lo(double v) { return __double2float_rd(v); }
__device__ __forceinline__ float box_hi(double v) { return __double2float_ru(v); }

// one thread per leaf: the bucket's box, then up the parent chain -- the second
// child to arrive at a node (atomic count) merges both boxes and continues
template <typename T>
__global__ void k_qboxes(const KdNode* __restrict__ nodes, int64_t nn, const T* __restrict__ coords, int64_t n,
                         int dims, QNode* __restrict__ qn, const int32_t* __restrict__ parent,
                         int32_t* __restrict__ arrive) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
    const KdNode rec = nodes[i];
    if (rec.db >= 0) return;
    int32_t c = (int32_t)i;
    int32_t p = parent[c];
    if (p < 0) return;  // the root is a leaf: no box needed
    float b[6];
#pragma unroll
    for (int d = 0; d < 3; d++) {
        float lo = INFINITY, hi = -INFINITY;
        if (d < dims) {
            const T* col = coords + (int64_t)d * n + rec.a;
            const int len = -1 - rec.db;
            for (int j = 0; j < len; j++) {
                const T v = col[j];
                lo = fminf(lo, box_lo(v));
                hi = fmaxf(hi, box_hi(v));
            }
        } else {
            lo = hi = 0.0f;
        }
        b[d] = lo;
        b[3 + d] = hi;
    }
    for (;;) {
        float* slot = (c == p + 1) ? qn[p].lb : qn[p].rb;
#pragma unroll
        for (int d = 0; d < 6; d++) slot[d] = b[d];
        __threadfence();
        if (atomicAdd(&arrive[p], 1) == 0) return;  // the sibling finishes this node
        __threadfence();
#pragma unroll
        for (int d = 0; d < 3; d++) {
            b[d] = fminf(__ldcg(&qn[p].lb[d]), __ldcg(&qn[p].rb[d]));
            b[3 + d] = fmaxf(__ldcg(&qn[p].lb[3 + d]), __ldcg(&qn[p].rb[3 + d]));
        }
        c = p;
        p = parent[p];
        if (p < 0) return;
    }
}

void build_qtree(KdTreeDev* t, cudaStream_t st) {
    if (t->dims > 3 || t->n_nodes < 1) return;
    const int64_t nn = t->n_nodes;
    KD_CUDA(cudaMallocAsync(&t->qnodes, nn * sizeof(QNode), st));
    int32_t *parent = nullptr, *arrive = nullptr;
    KD_CUDA(cudaMallocAsync((void**)&parent, nn * 4, st));
    KD_CUDA(cudaMallocAsync((void**)&arrive, nn * 4, st));
    KD_CUDA(cudaMemsetAsync(arrive, 0, nn * 4, st));
    const unsigned g = (unsigned)((nn + 255) / 256);
    k_qlinks<<<g, 256, 0, st>>>(t->nodes, nn, t->qnodes, parent);
    if (t->dtype == DT_F32)
        k_qboxes<float><<<g, 256, 0, st>>>(t->nodes, nn, (const float*)t->coords, t->n, t->dims, t->qnodes, parent,
                                           arrive);
    else
        k_qboxes<double><<<g, 256, 0, st>>>(t->nodes, nn, (const double*)t->coords, t->n, t->dims, t->qnodes,
                                            parent, arrive);
    KD_CUDA(cudaGetLastError());
    cudaFreeAsync(parent, st);
    cudaFreeAsync(arrive, st);
}

// ---------------------------------------------------------------------------
// the packet kernel
// ---------------------------------------------------------------------------
constexpr int PK_WARPS = 4;

template <typename T> struct PkPt { T c[4]; };

// squared distance from the query bracket [ql, qh] to a box, rounded down at
// every step: o_d = max(lo_d - qh_d, ql_d - hi_d, 0) (f32, round-down), then
// fma_rd(o_d, o_d, acc).  For every point p in the box and the binary64
// distance F(p) = RN(..RN(RN(a_0^2) + RN(a_1^2)) ..), a_d = RN(p_d - q_d):
// |a_d| >= o_d (monotone RN, o_d is an f32 <= |p_d - q_d|), RN(a_d^2) >= o_d^2
// (exact in binary64), and each RN sum >= the round-down f32 fma of smaller
// operands -- so the bound never exceeds F(p).
template <int DT>
__device__ __forceinline__ float box_bound(const float* __restrict__ b, const float (&ql)[3], const float (&qh)[3]) {
    float acc = 0.0f;
#pragma unroll
    for (int d = 0; d < DT; d++) {
        const float o = fmaxf(fmaxf(__fsub_rd(b[d], qh[d]), __fsub_rd(ql[d], b[3 + d])), 0.0f);
        acc = __fmaf_rd(o, o, acc);
    }
    return acc;
}

// the fp32 pre-filter threshold of kd_topk.cuh (f32_filter_thr) evaluated with
// round-up f32 steps: thr = (x + 2b + a sqrt(x + b)) * C, x = R (1 + 2^-22),
// a = 2u|q|, b = (u|q|)^2, C = (1 + (D+2)u) / (1-2u)^2 (1 + 1e-12), every input
// rounded up -- never below the binary64 expression, so still exact
__device__ __forceinline__ float thr_fast(double R, float a, float b, float C) {
    if (!(R < 1e30)) return INFINITY;
    const float x = __fmul_ru(__double2float_ru(R), 1.0000002384185791f);
    const float s = __fsqrt_ru(__fadd_ru(x, b));
    return __fmul_ru(__fadd_ru(__fadd_ru(x, __fmul_ru(2.0f, b)), __fmul_ru(a, s)), C);
}

template <typename T, int DT, int KM>
__global__ void __launch_bounds__(PK_WARPS * 32, (KM <= 8) ? 5 : 3)
k_knn_pkt(const QNode* __restrict__ qn, const KdNode* __restrict__ nodes, int32_t root_cnt,
          const T* __restrict__ coords, const uint64_t* __restrict__ ids, int64_t n,
          const double* __restrict__ queries, const int32_t* __restrict__ order, int64_t nq, int k,
          const double* __restrict__ radii, const uint64_t* __restrict__ excl, double* __restrict__ out_d,
          uint64_t* __restrict__ out_i, int64_t* __restrict__ out_c, int64_t* __restrict__ out_ctr,
          unsigned long long* __restrict__ counter, int cap) {
    constexpr bool F32 = sizeof(T) == 4;
    extern __shared__ __align__(16) unsigned char pk_dsmem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t per_warp = (size_t)cap * 32 * 4 + (size_t)cap * 8 + 32 * sizeof(PkPt<T>);
    unsigned char* base = pk_dsmem + warp * per_warp;
    PkPt<T>* s_p = reinterpret_cast<PkPt<T>*>(base);
    float* s_b = reinterpret_cast<float*>(base + 32 * sizeof(PkPt<T>));
    int2* s_r = reinterpret_cast<int2*>(s_b + (size_t)cap * 32);
    const bool has_ex = excl != nullptr;
    const int kk = k + (has_ex ? 1 : 0);  // top-(k+1) minus the excluded id, truncated to k
    const long long npk = (nq + 31) / 32;
    constexpr float U = 5.9604644775390625e-08f;
    const float CF = __fmul_ru(__fdiv_ru(1.0f + (DT + 2) * U, __fmul_rd(1.0f - 2.0f * U, 1.0f - 2.0f * U)),
                               1.0000001192092896f);

    for (;;) {
        long long pk = 0;
        if (lane == 0) pk = (long long)atomicAdd(counter, 1ULL);
        pk = __shfl_sync(FULL, pk, 0);
        if (pk >= npk) break;
        const int64_t t = pk * 32 + lane;
        const bool valid = t < nq;
        const int64_t qi = valid ? (order ? (int64_t)order[t] : t) : 0;
        double q[DT];
        float q32[DT], ql[3], qh[3];
        float qn2 = 0.0f;
#pragma unroll
        for (int d = 0; d < DT; d++) {
            q[d] = valid ? queries[qi * DT + d] : 0.0;
            q32[d] = __double2float_rn(q[d]);
            ql[d] = __double2float_rd(q[d]);
            qh[d] = __double2float_ru(q[d]);
            const float m = fmaxf(fabsf(ql[d]), fabsf(qh[d]));
            qn2 = __fmaf_ru(m, m, qn2);
        }
#pragma unroll
        for (int d = DT; d < 3; d++) ql[d] = qh[d] = 0.0f;
        const float uq = __fmul_ru(U, __fsqrt_ru(qn2));  // u|q|, rounded up
        const float fa = __fmul_ru(2.0f, uq), fb = __fmul_ru(uq, uq);
        const double radius = valid ? (radii ? radii[qi] : INFINITY) : -INFINITY;
        const uint64_t ex = (valid && has_ex) ? excl[qi] : ~0ULL;
        double bd[KM];
        uint32_t bp[KM];
#pragma unroll
        for (int j = 0; j < KM; j++) { bd[j] = INFINITY; bp[j] = 0; }
        int cnt = 0;
        double kth = radius;
        uint32_t kthp = 0;
        float thr32 = F32 ? thr_fast(radius, fa, fb, CF) : INFINITY;
        int c0 = 0, c1 = 0, c2 = 0;
        auto admit = [&](float b) { return valid && (cnt < kk ? (double)b < radius : (double)b <= kth); };

        // every active lane scans bucket [start, start + len), staged once in shared memory
        auto scan_leaf = [&](int start, int len, bool act) {
            c1 += act;
            c2 += act ? len : 0;
            for (int b0 = 0; b0 < len; b0 += 32) {
                const int m = min(32, len - b0);
                if (lane < m) {
                    PkPt<T> p;
#pragma unroll
                    for (int d = 0; d < 4; d++) p.c[d] = d < DT ? coords[(int64_t)d * n + start + b0 + lane] : T(0);
                    s_p[lane] = p;
                }
                __syncwarp();
                if (act) {
                    for (int j = 0; j < m; j++) {
                        const PkPt<T> p = s_p[j];
                        bool take = true;
                        if constexpr (F32) {
                            float d32 = 0.0f;
#pragma unroll
                            for (int d = 0; d < DT; d++) {
                                const float tt = (float)p.c[d] - q32[d];
                                d32 = fmaf(tt, tt, d32);
                            }
                            take = !(d32 > thr32);
                        }
                        if (take) {
                            double dist = 0.0;
#pragma unroll
                            for (int d = 0; d < DT; d++) {
                                const double df = __dsub_rn((double)p.c[d], q[d]);
                                dist = __dadd_rn(dist, __dmul_rn(df, df));
                            }
                            const uint32_t pos = (uint32_t)(start + b0 + j);
                            if (cnt < kk ? dist < radius : (dist <= kth && lexless_pos(dist, pos, kth, kthp, ids))) {
                                topk_insert_pos<KM>(bd, bp, cnt, kk, dist, pos, ids);
                                if (cnt == kk) {
                                    topk_last<KM>(bd, bp, kk, kth, kthp);
                                    if constexpr (F32) thr32 = thr_fast(kth, fa, fb, CF);
                                }
                            }
                        }
                    }
                }
                __syncwarp();
            }
        };

        // ---- phase 1: every lane's home leaf (descent by the split planes), then the
        // distinct home leaves of the packet scanned by all lanes -- every query starts the
        // shared walk with a k-th distance from its own neighbourhood
        int hs = 0, hl = 0;  // this lane's home bucket
        if (root_cnt < 0) {
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
            hs = rec.a;
            hl = -1 - rec.db;
        } else {
            hl = root_cnt;
        }
        int nh = 0;        // distinct home buckets scanned (lane j holds the j-th start in hstart)
        int hstart = -1;
        {
            bool pending = valid;
            unsigned mp;
            while ((mp = __ballot_sync(FULL, pending)) != 0) {
                const int src = __ffs(mp) - 1;
                const int s0 = __shfl_sync(FULL, hs, src), l0 = __shfl_sync(FULL, hl, src);
                if (lane == nh) hstart = s0;
                nh++;
                c0 += valid;
                scan_leaf(s0, l0, valid);
                if (pending && hs == s0) pending = false;
            }
        }

        // ---- phase 2: the shared depth-first walk
        int cref = 0, ccnt = root_cnt;
        float cb = 0.0f;
        int sp = 0;
        for (;;) {
            const bool act = admit(cb);
            if (__any_sync(FULL, act)) {
                if (ccnt >= 0) {
                    if (!__any_sync(FULL, lane < nh && hstart == cref)) {  // home buckets are done
                        c0 += act;
                        scan_leaf(cref, ccnt, act);
                    }
                } else {
                    // ---- interior: both children's boxes in one 64-byte record
                    const float4* r4 = reinterpret_cast<const float4*>(qn + cref);
                    const float4 v0 = __ldg(r4), v1 = __ldg(r4 + 1), v2 = __ldg(r4 + 2);
                    const int4 lk = __ldg(reinterpret_cast<const int4*>(r4 + 3));
                    const float lb[6] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y};
                    const float rb[6] = {v1.z, v1.w, v2.x, v2.y, v2.z, v2.w};
                    const float bl = box_bound<DT>(lb, ql, qh), br = box_bound<DT>(rb, ql, qh);
                    c0 += act;
                    const bool aL = act && admit(bl), aR = act && admit(br);
                    const unsigned mL = __ballot_sync(FULL, aL), mR = __ballot_sync(FULL, aR);
                    if (mL | mR) {
                        bool goL;
                        if (!mR) goL = true;
                        else if (!mL) goL = false;
                        else {
                            const unsigned vl = __ballot_sync(FULL, aL && (!aR || bl <= br));
                            const unsigned vr = __ballot_sync(FULL, aR && (!aL || br < bl));
                            goL = __popc(vl) >= __popc(vr);
                        }
                        const unsigned mfar = goL ? mR : mL;
                        if (mfar) {
                            if (sp >= cap) __trap();  // unreachable: at most one pushed entry per tree level
                            s_b[sp * 32 + lane] = goL ? br : bl;
                            if (lane == 0) s_r[sp] = goL ? make_int2(lk.z, lk.w) : make_int2(lk.x, lk.y);
                            sp++;
                        }
                        cref = goL ? lk.x : lk.z;
                        ccnt = goL ? lk.y : lk.w;
                        cb = goL ? bl : br;
                        continue;
                    }
                }
            }
            // ---- next subtree from the stack
            if (sp == 0) break;
            __syncwarp();
            sp--;
            const int2 e = s_r[sp];
            cref = e.x;
            ccnt = e.y;
            cb = s_b[sp * 32 + lane];
        }
        __syncwarp();
        if (valid) {
            int wr = 0;
            bool dropped = false;
#pragma unroll
            for (int j = 0; j < KM; j++) {
                if (j < cnt) {
                    const uint64_t id = ids[bp[j]];
                    if (has_ex && !dropped && id == ex) {
                        dropped = true;
                    } else if (wr < k) {
                        out_d[qi * (int64_t)k + wr] = bd[j];
                        out_i[qi * (int64_t)k + wr] = id;
                        wr++;
                    }
                }
            }
            out_c[qi] = wr;
            if (out_ctr) {
                out_ctr[qi * 3 + 0] = c0;
                out_ctr[qi * 3 + 1] = c1;
                out_ctr[qi * 3 + 2] = c2;
            }
        }
    }
}

static size_t pk_smem(int cap, size_t tsize) {
    return (size_t)PK_WARPS * ((size_t)cap * 32 * 4 + (size_t)cap * 8 + 32 * 4 * tsize);
}

template <typename T, int DT, int KM>
static void launch_pkt(const KdTreeDev& t, const KnnArgs& a, const int32_t* order, cudaStream_t st) {
    const int cap = (int)((std::max<int64_t>(t.depth + 2, 4) + 1) & ~1LL);  // even: 16-byte aligned warp slices
    const size_t smem = pk_smem(cap, sizeof(T));
    auto kern = k_knn_pkt<T, DT, KM>;
    KD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 148, per_sm = 0;
    KD_CUDA(cudaGetDevice(&dev));
    KD_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    KD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PK_WARPS * 32, smem));
    const long long packets = (a.nq + 31) / 32;
    const long long want = (packets + PK_WARPS - 1) / PK_WARPS;
    const unsigned grid = (unsigned)std::max(1LL, std::min<long long>(want, (long long)sms * std::max(per_sm, 1)));
    unsigned long long* ctr = nullptr;
    KD_CUDA(cudaMallocAsync((void**)&ctr, sizeof(unsigned long long), st));
    KD_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
    // the root as a child reference: interior node 0, or (a one-node tree) the whole tree as one bucket
    const int32_t root_cnt = t.n_nodes == 1 ? (int32_t)t.n : -1;
    kern<<<grid, PK_WARPS * 32, smem, st>>>(static_cast<const QNode*>(t.qnodes), t.nodes, root_cnt,
                                            static_cast<const T*>(t.coords), t.ids, t.n, a.queries, order, a.nq,
                                            (int)a.k, a.radii, a.excl, a.out_d, a.out_i, a.out_c, a.out_ctr, ctr, cap);
    KD_CUDA(cudaGetLastError());
    cudaFreeAsync(ctr, st);
}

template <typename T, int DT>
static bool pkt_k(const KdTreeDev& t, const KnnArgs& a, const int32_t* order, cudaStream_t st) {
    const int64_t kc = a.k + (a.excl ? 1 : 0);
    if (kc == 1) launch_pkt<T, DT, 1>(t, a, order, st);
    else if (kc == 2) launch_pkt<T, DT, 2>(t, a, order, st);
    else if (kc <= 4) launch_pkt<T, DT, 4>(t, a, order, st);
    else if (kc <= 6) launch_pkt<T, DT, 6>(t, a, order, st);
    else if (kc <= 8) launch_pkt<T, DT, 8>(t, a, order, st);
    else if (kc <= 16) launch_pkt<T, DT, 16>(t, a, order, st);
    else if (kc <= 32) launch_pkt<T, DT, 32>(t, a, order, st);
    else return false;
    return true;
}

bool knn_packet(const KdTreeDev& t, const KnnArgs& a, const int32_t* order, cudaStream_t st) {
    if (!t.qnodes || t.dims < 1 || t.dims > 3 || a.thread_per_query || !a.packet) return false;
    if (a.k + (a.excl ? 1 : 0) > 32) return false;
    const bool f32 = t.dtype == DT_F32;
    switch (t.dims) {
        case 1: return f32 ? pkt_k<float, 1>(t, a, order, st) : pkt_k<double, 1>(t, a, order, st);
        case 2: return f32 ? pkt_k<float, 2>(t, a, order, st) : pkt_k<double, 2>(t, a, order, st);
        default: return f32 ? pkt_k<float, 3>(t, a, order, st) : pkt_k<double, 3>(t, a, order, st);
    }
}

}  // namespace kdb
