// kd_dist.cu -- device kernels of the global (multi-GPU) tier.  Every entry point
// only enqueues work on the caller's stream (no host synchronisation): results
// that the protocol needs on the host (histograms, counts) travel through the
// caller's collectives first and are read back once per exchange.
//
//   kd_histogram   counts / equals of one coordinate row against sorted boundaries
//                  (median.py:128-140 histogram_with_equals; cluster.py:246)
//   kd_split_rows  stable two-way split of a rank's SoA points by a plane, low side
//                  first (cluster.py:292-294), written as packed AoS rows -- the
//                  all-to-all send buffer of the redistribution (cluster.py:302-346)
//   kd_unpack_rows packed rows back to SoA coordinates + ids
//   kd_route       owner rank of each query (cluster.py:96-114, ties right) and
//                  the bitmask of other ranks whose region is strictly within
//                  the query's squared radius (cluster.py:133-154)
//   kd_merge_topk  owner-side merge of the local top-k and the remote replies by
//                  (sq_dist, point_id) (dist_query.py:138-161), duplicate ids flagged
// Binary64 comparisons throughout, identical to the reference's arithmetic.
#include <cub/cub.cuh>

#include <string>

#include "../../include/kdtree_b200.h"
#include "kd_arena.cuh"
#include "kd_common.cuh"

namespace kdb {

constexpr int HIST_THREADS = 256;
constexpr int HIST_MAXB = 4096;

template <typename T>
__global__ void __launch_bounds__(HIST_THREADS)
k_hist_full(const T* __restrict__ v, int64_t n, const double* __restrict__ b, int nb,
            unsigned long long* __restrict__ counts, unsigned long long* __restrict__ equals) {
    extern __shared__ __align__(16) unsigned char hsm[];
    double* sb = reinterpret_cast<double*>(hsm);
    unsigned int* sc = reinterpret_cast<unsigned int*>(sb + nb);
    unsigned int* se = sc + nb + 1;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) { sb[i] = b[i]; se[i] = 0; }
    for (int i = threadIdx.x; i <= nb; i += blockDim.x) sc[i] = 0;
    __syncthreads();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = (double)v[i];
        int lo = 0, hi = nb;  // number of boundaries <= x (median.py:99 _locate)
        while (lo < hi) {
            const int md = (lo + hi) >> 1;
            if (sb[md] <= x) lo = md + 1; else hi = md;
        }
        atomicAdd(&sc[lo], 1u);
        if (lo > 0 && sb[lo - 1] == x) atomicAdd(&se[lo - 1], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= nb; i += blockDim.x)
        if (sc[i]) atomicAdd(&counts[i], (unsigned long long)sc[i]);
    if (equals)
        for (int i = threadIdx.x; i < nb; i += blockDim.x)
            if (se[i]) atomicAdd(&equals[i], (unsigned long long)se[i]);
}

template <typename T>
__global__ void k_flag_low(const T* __restrict__ row, int64_t n, double value, int32_t* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (double)row[i] < value ? 1 : 0;
}

__global__ void k_count_low(const int32_t* __restrict__ flag, const int32_t* __restrict__ pre, int64_t n,
                            int64_t* __restrict__ n_low) {
    n_low[0] = n ? (int64_t)pre[n - 1] + flag[n - 1] : 0;
}

// packed row: dims coordinates (storage type), padded to 8 bytes, then the 8-byte id
__host__ __device__ inline int row_bytes(int dims, int es) { return ((dims * es + 7) & ~7) + 8; }

template <typename T>
__global__ void k_split_scatter(const T* __restrict__ coords, const uint64_t* __restrict__ ids, int64_t n, int dims,
                                const int32_t* __restrict__ flag, const int32_t* __restrict__ pre,
                                const int64_t* __restrict__ n_low, unsigned char* __restrict__ rows) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t nl = n_low[0];
    const int64_t p = flag[i] ? (int64_t)pre[i] : nl + (i - pre[i]);
    const int W = row_bytes(dims, (int)sizeof(T));
    unsigned char* r = rows + p * W;
    for (int d = 0; d < dims; d++) reinterpret_cast<T*>(r)[d] = coords[(int64_t)d * n + i];
    *reinterpret_cast<uint64_t*>(r + W - 8) = ids[i];
}

template <typename T>
__global__ void k_unpack(const unsigned char* __restrict__ rows, int64_t n, int dims, T* __restrict__ coords,
                         uint64_t* __restrict__ ids) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int W = row_bytes(dims, (int)sizeof(T));
    const unsigned char* r = rows + i * W;
    for (int d = 0; d < dims; d++) coords[(int64_t)d * n + i] = reinterpret_cast<const T*>(r)[d];
    ids[i] = *reinterpret_cast<const uint64_t*>(r + W - 8);
}

__global__ void k_route(const int32_t* __restrict__ pdim, const double* __restrict__ pval, int P,
                        const double* __restrict__ lo, const double* __restrict__ hi, const double* __restrict__ q,
                        int64_t nq, int dims, const double* __restrict__ radii, int32_t* __restrict__ owner,
                        unsigned long long* __restrict__ within) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nq) return;
    const double* qq = q + i * dims;
    int idx = 0;
    const int np = P - 1;
    while (idx < np) {
        const int bit = qq[pdim[idx]] < pval[idx] ? 0 : 1;
        idx = 2 * idx + 1 + bit;
    }
    const int own = idx - np;
    if (owner) owner[i] = own;
    if (within) {
        const double r = radii ? radii[i] : INFINITY;
        unsigned long long m = 0ULL;
        for (int rk = 0; rk < P; rk++) {
            if (rk == own) continue;
            double s = 0.0;  // core.py:231-244 min_sq_dist_to_region
            for (int d = 0; d < dims; d++) {
                const double qd = qq[d], l = lo[rk * dims + d], h = hi[rk * dims + d];
                double o = 0.0;
                if (qd < l) o = __dsub_rn(l, qd);
                else if (qd > h) o = __dsub_rn(qd, h);
                s = __dadd_rn(s, __dmul_rn(o, o));
            }
            if (s < r) m |= 1ULL << rk;
        }
        within[i] = m;
    }
}

// ---- owner-side merge -------------------------------------------------------
__global__ void k_merge_count(const int64_t* __restrict__ slot, int64_t nr, int32_t* __restrict__ cnt) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nr) atomicAdd(&cnt[slot[t]], 1);
}
__global__ void k_merge_fill(const int64_t* __restrict__ slot, int64_t nr, const int32_t* __restrict__ start,
                             int32_t* __restrict__ fillc, int32_t* __restrict__ list) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < nr) {
        const int64_t j = slot[t];
        list[start[j] + atomicAdd(&fillc[j], 1)] = (int32_t)t;
    }
}

constexpr int MERGE_MAXL = 65;  // own list + at most 64 ranks' replies

// one thread per owned query: k-way merge of its sorted candidate lists by (d, id);
// the merge runs over every candidate so that a duplicate id anywhere in the pool is
// seen (equal ids from one point have equal distances, so they are adjacent)
__global__ void k_merge(int64_t m, int k, const double* __restrict__ ld, const uint64_t* __restrict__ li,
                        const int64_t* __restrict__ lc, int32_t my_rank, const double* __restrict__ rd,
                        const uint64_t* __restrict__ ri, const int64_t* __restrict__ rc,
                        const int32_t* __restrict__ rrank, const int32_t* __restrict__ start,
                        const int32_t* __restrict__ cnt, const int32_t* __restrict__ list, double* __restrict__ od,
                        uint64_t* __restrict__ oi, int32_t* __restrict__ orank, int64_t* __restrict__ oc,
                        int32_t* __restrict__ dup) {
    const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int nl = 1 + (cnt ? min(cnt[j], MERGE_MAXL - 1) : 0);
    int row[MERGE_MAXL];
    int pos[MERGE_MAXL];
    int len[MERGE_MAXL];
    row[0] = -1;
    pos[0] = 0;
    len[0] = (int)lc[j];
    for (int l = 1; l < nl; l++) {
        row[l] = list[start[j] + l - 1];
        pos[l] = 0;
        len[l] = (int)rc[row[l]];
    }
    int w = 0;
    double last_d = -1.0;
    uint64_t last_i = 0;
    bool have_last = false;
    for (;;) {
        int best = -1;
        double bd = 0.0;
        uint64_t bi = 0;
        for (int l = 0; l < nl; l++) {
            if (pos[l] >= len[l]) continue;
            const int64_t e = (row[l] < 0 ? j : (int64_t)row[l]) * k + pos[l];
            const double d = row[l] < 0 ? ld[e] : rd[e];
            const uint64_t id = row[l] < 0 ? li[e] : ri[e];
            if (best < 0 || d < bd || (d == bd && id < bi)) {
                best = l;
                bd = d;
                bi = id;
            }
        }
        if (best < 0) break;
        if (have_last && bi == last_i && bd == last_d) atomicExch(dup, 1);
        have_last = true;
        last_d = bd;
        last_i = bi;
        if (w < k) {
            od[j * k + w] = bd;
            oi[j * k + w] = bi;
            orank[j * k + w] = row[best] < 0 ? my_rank : rrank[row[best]];
            w++;
        }
        pos[best]++;
    }
    oc[j] = w;
}

int derr(int code, const std::string& m);

}  // namespace kdb

// error plumbing shared with kd_capi.cu (thread-local kd_last_error message)
int kd_set_error(int code, const char* msg);
int kdb::derr(int code, const std::string& m) { return kd_set_error(code, m.c_str()); }

using namespace kdb;

#define KD_DTRY(...)                                                   \
    try {                                                              \
        __VA_ARGS__;                                                   \
    } catch (const kdb::CudaError& e) {                                \
        return derr(KD_ECUDA, e.msg);                                  \
    } catch (const std::exception& e) {                                \
        return derr(KD_ECUDA, e.what());                               \
    }

static int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

extern "C" {

KD_API int kd_histogram(const void* values, int dtype, int64_t n, const double* boundaries, int64_t nb,
                        int64_t* counts, int64_t* equals, unsigned flags, void* stream) {
    if (nb < 1 || nb > HIST_MAXB) return derr(KD_EUNSUPPORTED, "kd_histogram: nb must be in [1, 4096]");
    if (n < 0) return derr(KD_EINVAL, "kd_histogram: n < 0");
    if (dtype != KD_F32 && dtype != KD_F64) return derr(KD_EINVAL, "kd_histogram: bad dtype");
    if (!counts) return derr(KD_EINVAL, "kd_histogram: counts is NULL");
    KD_DTRY({
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const bool dp = flags & KD_DEVICE_PTRS;
        const size_t es = dtype == KD_F32 ? 4 : 8;
        StreamArena sa(current_device(), st);
        const void* v = values;
        const double* b = boundaries;
        unsigned long long* dc = reinterpret_cast<unsigned long long*>(counts);
        unsigned long long* de = reinterpret_cast<unsigned long long*>(equals);
        if (!dp) {
            void* dv = scratch<unsigned char>(n * es, st);
            double* db = scratch<double>(nb, st);
            if (n) KD_CUDA(cudaMemcpyAsync(dv, values, n * es, cudaMemcpyHostToDevice, st));
            KD_CUDA(cudaMemcpyAsync(db, boundaries, nb * 8, cudaMemcpyHostToDevice, st));
            v = dv;
            b = db;
            dc = scratch<unsigned long long>(nb + 1, st);
            de = equals ? scratch<unsigned long long>(nb, st) : nullptr;
        }
        KD_CUDA(cudaMemsetAsync(dc, 0, (nb + 1) * 8, st));
        if (de) KD_CUDA(cudaMemsetAsync(de, 0, nb * 8, st));
        if (n) {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, current_device());
            const unsigned grid = (unsigned)std::min<int64_t>((n + HIST_THREADS - 1) / HIST_THREADS, (int64_t)sms * 4);
            const size_t sm = (size_t)nb * 8 + (size_t)(nb + 1) * 4 + (size_t)nb * 4;
            KD_CUDA(cudaFuncSetAttribute(k_hist_full<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000));
            KD_CUDA(cudaFuncSetAttribute(k_hist_full<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000));
            if (dtype == KD_F32)
                k_hist_full<float><<<grid, HIST_THREADS, sm, st>>>((const float*)v, n, b, (int)nb, dc, de);
            else
                k_hist_full<double><<<grid, HIST_THREADS, sm, st>>>((const double*)v, n, b, (int)nb, dc, de);
            KD_CUDA(cudaGetLastError());
        }
        if (!dp) {  // host outputs: the one synchronous mode
            KD_CUDA(cudaMemcpyAsync(counts, dc, (nb + 1) * 8, cudaMemcpyDeviceToHost, st));
            if (equals) KD_CUDA(cudaMemcpyAsync(equals, de, nb * 8, cudaMemcpyDeviceToHost, st));
            KD_CUDA(cudaStreamSynchronize(st));
        }
    });
    return KD_OK;
}

KD_API int kd_split_rows(const void* coords, int dtype, int64_t n, int dims, const uint64_t* ids, int dim,
                         double value, void* out_rows, int64_t* n_low, unsigned flags, void* stream) {
    if (!(flags & KD_DEVICE_PTRS)) return derr(KD_EINVAL, "kd_split_rows: device pointers required");
    if (dims < 1 || dims > 16) return derr(KD_EINVAL, "kd_split_rows: dims out of range");
    if (dim < 0 || dim >= dims) return derr(KD_EINVAL, "kd_split_rows: dim out of range");
    if (dtype != KD_F32 && dtype != KD_F64) return derr(KD_EINVAL, "kd_split_rows: bad dtype");
    if (!n_low) return derr(KD_EINVAL, "kd_split_rows: n_low is NULL");
    if (n < 0 || n >= (int64_t(1) << 31)) return derr(KD_EUNSUPPORTED, "kd_split_rows: n must be in [0, 2^31)");
    KD_DTRY({
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (n == 0) {
            KD_CUDA(cudaMemsetAsync(n_low, 0, 8, st));
            return KD_OK;
        }
        StreamArena sa(current_device(), st);
        int32_t* fl = scratch<int32_t>(n, st);
        int32_t* pre = scratch<int32_t>(n, st);
        const unsigned g = (unsigned)((n + 255) / 256);
        const size_t es = dtype == KD_F32 ? 4 : 8;
        const char* row = static_cast<const char*>(coords) + (size_t)dim * n * es;
        if (dtype == KD_F32) k_flag_low<float><<<g, 256, 0, st>>>((const float*)row, n, value, fl);
        else k_flag_low<double><<<g, 256, 0, st>>>((const double*)row, n, value, fl);
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, fl, pre, (int)n, st);
        void* tmp = scratch<unsigned char>(tb, st);
        cub::DeviceScan::ExclusiveSum(tmp, tb, fl, pre, (int)n, st);
        k_count_low<<<1, 1, 0, st>>>(fl, pre, n, n_low);
        if (dtype == KD_F32)
            k_split_scatter<float><<<g, 256, 0, st>>>((const float*)coords, ids, n, dims, fl, pre, n_low,
                                                     (unsigned char*)out_rows);
        else
            k_split_scatter<double><<<g, 256, 0, st>>>((const double*)coords, ids, n, dims, fl, pre, n_low,
                                                      (unsigned char*)out_rows);
        KD_CUDA(cudaGetLastError());
    });
    return KD_OK;
}

KD_API int kd_unpack_rows(const void* rows, int64_t n, int dims, int dtype, void* out_coords, uint64_t* out_ids,
                          unsigned flags, void* stream) {
    if (!(flags & KD_DEVICE_PTRS)) return derr(KD_EINVAL, "kd_unpack_rows: device pointers required");
    if (dims < 1 || dims > 16) return derr(KD_EINVAL, "kd_unpack_rows: dims out of range");
    if (dtype != KD_F32 && dtype != KD_F64) return derr(KD_EINVAL, "kd_unpack_rows: bad dtype");
    if (n <= 0) return KD_OK;
    KD_DTRY({
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const unsigned g = (unsigned)((n + 255) / 256);
        if (dtype == KD_F32)
            k_unpack<float><<<g, 256, 0, st>>>((const unsigned char*)rows, n, dims, (float*)out_coords, out_ids);
        else
            k_unpack<double><<<g, 256, 0, st>>>((const unsigned char*)rows, n, dims, (double*)out_coords, out_ids);
        KD_CUDA(cudaGetLastError());
    });
    return KD_OK;
}

KD_API int kd_route(const int32_t* plane_dims, const double* plane_values, int32_t ranks, const double* region_lo,
                    const double* region_hi, const double* queries, int64_t nq, int dims, const double* radii,
                    int32_t* owner, uint64_t* within, unsigned flags, void* stream) {
    if (!(flags & KD_DEVICE_PTRS)) return derr(KD_EINVAL, "kd_route: device pointers required");
    if (ranks < 1 || ranks > 64 || (ranks & (ranks - 1))) return derr(KD_EINVAL, "kd_route: ranks must be a power of two <= 64");
    if (nq == 0) return KD_OK;
    KD_DTRY({
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        k_route<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(plane_dims, plane_values, ranks, region_lo, region_hi,
                                                              queries, nq, dims, radii, owner,
                                                              (unsigned long long*)within);
        KD_CUDA(cudaGetLastError());
    });
    return KD_OK;
}

KD_API int kd_merge_topk(int64_t m, int64_t k, const double* local_d, const uint64_t* local_i, const int64_t* local_c,
                         int32_t my_rank, int64_t nr, const int64_t* reply_slot, const double* reply_d,
                         const uint64_t* reply_i, const int64_t* reply_c, const int32_t* reply_rank, double* out_d,
                         uint64_t* out_i, int32_t* out_rank, int64_t* out_c, int32_t* dup_flag, unsigned flags,
                         void* stream) {
    if (!(flags & KD_DEVICE_PTRS)) return derr(KD_EINVAL, "kd_merge_topk: device pointers required");
    if (k < 1) return derr(KD_EINVAL, "kd_merge_topk: k must be >= 1");
    if (m <= 0) return KD_OK;
    if (m >= (int64_t(1) << 31) || nr >= (int64_t(1) << 31)) return derr(KD_EUNSUPPORTED, "kd_merge_topk: sizes >= 2^31");
    KD_DTRY({
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        StreamArena sa(current_device(), st);
        int32_t *cnt = nullptr, *start = nullptr, *list = nullptr;
        if (nr > 0) {
            cnt = scratch<int32_t>(m, st);
            start = scratch<int32_t>(m, st);
            int32_t* fillc = scratch<int32_t>(m, st);
            list = scratch<int32_t>(nr, st);
            KD_CUDA(cudaMemsetAsync(cnt, 0, m * 4, st));
            KD_CUDA(cudaMemsetAsync(fillc, 0, m * 4, st));
            const unsigned gr = (unsigned)((nr + 255) / 256);
            k_merge_count<<<gr, 256, 0, st>>>(reply_slot, nr, cnt);
            size_t tb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, start, (int)m, st);
            void* tmp = scratch<unsigned char>(tb, st);
            cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, start, (int)m, st);
            k_merge_fill<<<gr, 256, 0, st>>>(reply_slot, nr, start, fillc, list);
        }
        k_merge<<<(unsigned)((m + 127) / 128), 128, 0, st>>>(m, (int)k, local_d, local_i, local_c, my_rank, reply_d,
                                                             reply_i, reply_c, reply_rank, start, cnt, list, out_d,
                                                             out_i, out_rank, out_c, dup_flag);
        KD_CUDA(cudaGetLastError());
    });
    return KD_OK;
}

}  // extern "C"
