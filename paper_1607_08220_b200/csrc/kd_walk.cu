// kd_walk.cu -- depth-independent KNN walk with the reference's own traversal as an option.
//
// One thread per query, traversal stack and bounded max-heap in global scratch
// sized from the tree depth (cap = depth + 2, local_query.py:83-86) and k, so it
// serves
//   * REF = true  (KD_KNN_REFERENCE): Algorithm 1 exactly as local_query.py:72-172
//     walks it -- binary64 incremental bounds (bound - old_off^2 + new_off^2),
//     interior nodes pruned at bound >= r', far child pushed iff far_bound < r',
//     leaves never bound-checked, the reference's heap admission.  Results AND
//     the (nodes visited, buckets scanned, points compared) counters are
//     bit-identical to find_knn_batch of the reference, including its tie quirk
//     (SURVEY.md §8(a) Q5).
//   * REF = false: the same walk with the brute-force oracle's tie semantics
//     (prune only at bound > k-th distance; bounds re-summed with round-down
//     steps so they never exceed a true distance) for trees deeper than the
//     fixed stack of the fast kernels (kd_query.cu, KNN_MAX_DEPTH).
// Stack / heap layout: [entry][field][thread of the chunk] -> coalesced.
#include <algorithm>

#include "kd_arena.cuh"
#include "kd_common.cuh"
#include "kd_query.cuh"
#include "kd_topk.cuh"
#include "kd_tree.cuh"

namespace kdb {

constexpr int WALK_DMAX = 16;
constexpr int WALK_THREADS = 128;

template <typename T, bool REF>
__global__ void __launch_bounds__(WALK_THREADS)
k_knn_walk(const KdNode* __restrict__ nodes, int64_t n_nodes, const T* __restrict__ coords,
           const uint64_t* __restrict__ ids, int64_t n, int D, const double* __restrict__ queries, int64_t q0,
           int64_t cnt_q, int k, const double* __restrict__ radii, const uint64_t* __restrict__ excl,
           double* __restrict__ out_d, uint64_t* __restrict__ out_i, int64_t* __restrict__ out_c,
           int64_t* __restrict__ out_ctr, int32_t* __restrict__ st_node, double* __restrict__ st_bound,
           double* __restrict__ st_off, double* __restrict__ hd, uint64_t* __restrict__ hi, int64_t CT) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= cnt_q) return;
    const int64_t qi = q0 + t;
    double q[WALK_DMAX], cur[WALK_DMAX];
#pragma unroll
    for (int d = 0; d < WALK_DMAX; d++) q[d] = d < D ? queries[qi * D + d] : 0.0;
    const double radius = radii ? radii[qi] : INFINITY;
    const bool has_ex = !REF && excl != nullptr;
    const uint64_t ex = has_ex ? excl[qi] : 0ULL;
    int64_t c0 = 0, c1 = 0, c2 = 0;
    double r_prime = radius;  // local_query.py:96: the radius while under-full, the heap's max distance when full
    int hs = 0;
    auto H_d = [&](int j) -> double& { return hd[(int64_t)j * CT + t]; };
    auto H_i = [&](int j) -> uint64_t& { return hi[(int64_t)j * CT + t]; };
    auto heap_less = [&](int a, int b) { return lexless(H_d(a), H_i(a), H_d(b), H_i(b)); };
    auto heap_swap = [&](int a, int b) {
        const double td = H_d(a); H_d(a) = H_d(b); H_d(b) = td;
        const uint64_t ti = H_i(a); H_i(a) = H_i(b); H_i(b) = ti;
    };
    auto sift_down = [&](int size) {  // local_query.py:52-69 _heap_replace_root after the root was overwritten
        int i = 0;
        for (;;) {
            const int l = 2 * i + 1, r = l + 1;
            int big = i;
            if (l < size && heap_less(big, l)) big = l;
            if (r < size && heap_less(big, r)) big = r;
            if (big == i) break;
            heap_swap(big, i);
            i = big;
        }
    };
    // admissible(bound): may the subtree still hold a neighbour?  REF prunes at bound >= r'
    auto admissible = [&](double b) { return REF ? b < r_prime : (hs < k ? b < r_prime : b <= r_prime); };

    int sp = 0;
    if (n_nodes > 0) {
        st_node[t] = 0;
        st_bound[t] = 0.0;
        for (int d = 0; d < D; d++) st_off[(int64_t)d * CT + t] = 0.0;
        sp = 1;
    }
    while (sp > 0) {
        sp--;
        const int node = st_node[(int64_t)sp * CT + t];
        const double bound = st_bound[(int64_t)sp * CT + t];
#pragma unroll
        for (int d = 0; d < WALK_DMAX; d++)
            if (d < D) cur[d] = st_off[((int64_t)sp * D + d) * CT + t];
        c0++;
        const KdNode rec = nodes[node];
        if (rec.db < 0) {  // leaf: never bound-checked (local_query.py:114)
            const int start = rec.a, len = -1 - rec.db;
            c1++;
            c2 += len;
            for (int i = start; i < start + len; i++) {
                double dist = 0.0;
#pragma unroll
                for (int d = 0; d < WALK_DMAX; d++) {
                    if (d < D) {
                        const double df = __dsub_rn((double)coords[(int64_t)d * n + i], q[d]);
                        dist = __dadd_rn(dist, __dmul_rn(df, df));
                    }
                }
                if (hs < k) {
                    if (!(dist < r_prime)) continue;
                    const uint64_t id = ids[i];
                    if (has_ex && id == ex) continue;
                    int ii = hs;  // local_query.py:36-49 _heap_push
                    H_d(ii) = dist;
                    H_i(ii) = id;
                    while (ii > 0) {
                        const int pp = (ii - 1) / 2;
                        if (!heap_less(pp, ii)) break;
                        heap_swap(pp, ii);
                        ii = pp;
                    }
                    hs++;
                    if (hs == k) r_prime = H_d(0);
                } else {
                    if (!(dist <= r_prime)) continue;
                    const uint64_t id = ids[i];
                    if (has_ex && id == ex) continue;
                    if (!lexless(dist, id, H_d(0), H_i(0))) continue;
                    H_d(0) = dist;
                    H_i(0) = id;
                    sift_down(hs);
                    r_prime = H_d(0);
                }
            }
            continue;
        }
        if (!admissible(bound)) continue;  // local_query.py:136
        const int dim = rec.db;
        double qd = q[0], old_off = cur[0];
#pragma unroll
        for (int d = 1; d < WALK_DMAX; d++)
            if (d == dim) { qd = q[d]; old_off = cur[d]; }
        // REF: the reference's rounding; otherwise toward zero, so the offset never exceeds the true one
        const double new_off = REF ? __dsub_rn(qd, rec.v) : __dsub_rz(qd, rec.v);
        const bool goleft = qd < rec.v;
        const int near = goleft ? node + 1 : rec.a;
        const int far = goleft ? rec.a : node + 1;
        double far_bound;
        if (REF) {  // local_query.py:149: bound - old_off * old_off + new_off * new_off, left to right
            far_bound = __dadd_rn(__dsub_rn(bound, __dmul_rn(old_off, old_off)), __dmul_rn(new_off, new_off));
        } else {  // re-summed, every step rounded down: <= the distance of any point of the far box
            far_bound = 0.0;
#pragma unroll
            for (int d = 0; d < WALK_DMAX; d++)
                if (d < D) {
                    const double o = d == dim ? new_off : cur[d];
                    far_bound = __dadd_rd(far_bound, __dmul_rd(fabs(o), fabs(o)));
                }
        }
        if (admissible(far_bound)) {  // local_query.py:150
            st_node[(int64_t)sp * CT + t] = far;
            st_bound[(int64_t)sp * CT + t] = far_bound;
#pragma unroll
            for (int d = 0; d < WALK_DMAX; d++)
                if (d < D) st_off[((int64_t)sp * D + d) * CT + t] = d == dim ? new_off : cur[d];
            sp++;
        }
        st_node[(int64_t)sp * CT + t] = near;  // near child last: processed first
        st_bound[(int64_t)sp * CT + t] = bound;
#pragma unroll
        for (int d = 0; d < WALK_DMAX; d++)
            if (d < D) st_off[((int64_t)sp * D + d) * CT + t] = cur[d];
        sp++;
    }
    // drain max-first into the tail -> ascending (dist, id) (local_query.py:162-171)
    out_c[qi] = hs;
    int j = hs, size = hs;
    while (size > 0) {
        j--;
        out_d[qi * (int64_t)k + j] = H_d(0);
        out_i[qi * (int64_t)k + j] = H_i(0);
        size--;
        if (size > 0) {
            H_d(0) = H_d(size);
            H_i(0) = H_i(size);
            sift_down(size);
        }
    }
    if (out_ctr) {
        out_ctr[qi * 3 + 0] = c0;
        out_ctr[qi * 3 + 1] = c1;
        out_ctr[qi * 3 + 2] = c2;
    }
}

// queries per launch: bounds the scratch (stack + heap) to about 256 MB
static int64_t walk_chunk(const KdTreeDev& t, int64_t k, int64_t nq) {
    const int64_t cap = t.depth + 2;
    const int64_t per_q = cap * (4 + 8 + 8 * (int64_t)t.dims) + k * 16;
    int64_t c = std::max<int64_t>(WALK_THREADS, ((int64_t)256 << 20) / std::max<int64_t>(per_q, 1));
    c = (c / WALK_THREADS) * WALK_THREADS;
    return std::min(c, ((nq + WALK_THREADS - 1) / WALK_THREADS) * WALK_THREADS);
}

template <typename T>
static void walk_typed(const KdTreeDev& t, const KnnArgs& a, bool ref, cudaStream_t st) {
    const int64_t cap = t.depth + 2;
    const int64_t CT = walk_chunk(t, a.k, a.nq);
    int32_t* st_node = scratch<int32_t>((size_t)(cap * CT), st);
    double* st_bound = scratch<double>((size_t)(cap * CT), st);
    double* st_off = scratch<double>((size_t)(cap * CT * t.dims), st);
    double* hd = scratch<double>((size_t)(a.k * CT), st);
    uint64_t* hi = scratch<uint64_t>((size_t)(a.k * CT), st);
    for (int64_t q0 = 0; q0 < a.nq; q0 += CT) {
        const int64_t cnt = std::min(CT, a.nq - q0);
        const unsigned blocks = (unsigned)((cnt + WALK_THREADS - 1) / WALK_THREADS);
        if (ref)
            k_knn_walk<T, true><<<blocks, WALK_THREADS, 0, st>>>(
                t.nodes, t.n_nodes, (const T*)t.coords, t.ids, t.n, t.dims, a.queries, q0, cnt, (int)a.k, a.radii, a.excl,
                a.out_d, a.out_i, a.out_c, a.out_ctr, st_node, st_bound, st_off, hd, hi, CT);
        else
            k_knn_walk<T, false><<<blocks, WALK_THREADS, 0, st>>>(
                t.nodes, t.n_nodes, (const T*)t.coords, t.ids, t.n, t.dims, a.queries, q0, cnt, (int)a.k, a.radii, a.excl,
                a.out_d, a.out_i, a.out_c, a.out_ctr, st_node, st_bound, st_off, hd, hi, CT);
        KD_CUDA(cudaGetLastError());
    }
    scratch_free(st_node, st); scratch_free(st_bound, st); scratch_free(st_off, st);
    scratch_free(hd, st); scratch_free(hi, st);
}

void knn_walk(const KdTreeDev& t, const KnnArgs& a, bool reference, cudaStream_t st) {
    if (a.nq == 0) return;
    StreamArena ka(t.device, st);
    if (t.dtype == DT_F32) walk_typed<float>(t, a, reference, st);
    else walk_typed<double>(t, a, reference, st);
}

}  // namespace kdb
