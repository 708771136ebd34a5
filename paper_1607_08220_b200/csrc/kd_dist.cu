// kd_dist.cu -- device kernels of the global (multi-GPU) tier.
//
//   kd_histogram  : counts/equals of one coordinate row against sorted boundaries
//                   (median.py:128-140 histogram_with_equals; cluster.py:246)
//   kd_partition  : stable two-way split of a rank's points by a plane, low side
//                   first (cluster.py:292-294 side_idx, order preserved)
//   kd_route      : owner rank of each query (cluster.py:96-114, ties right) and
//                   the bitmask of other ranks whose region is strictly within
//                   the query's squared radius (cluster.py:133-154)
// Binary64 comparisons throughout, identical to the reference's arithmetic.
#include <cub/cub.cuh>

#include <string>

#include "../../include/kdtree_b200.h"
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
        int lo = 0, hi = nb;  // number of boundaries <= x
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
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
        if (se[i]) atomicAdd(&equals[i], (unsigned long long)se[i]);
}

template <typename T>
__global__ void k_flag_low(const T* __restrict__ row, int64_t n, double value, int32_t* __restrict__ flag) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) flag[i] = (double)row[i] < value ? 1 : 0;
}

template <typename T>
__global__ void k_part_scatter(const T* __restrict__ coords, const uint64_t* __restrict__ ids, int64_t n, int dims,
                               const int32_t* __restrict__ flag, const int64_t* __restrict__ pre, int64_t nlow,
                               T* __restrict__ oc, uint64_t* __restrict__ oi) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t p = flag[i] ? pre[i] : nlow + (i - pre[i]);
    for (int d = 0; d < dims; d++) oc[(int64_t)d * n + p] = coords[(int64_t)d * n + i];
    oi[p] = ids[i];
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

}  // namespace kdb

using namespace kdb;

// error plumbing shared with kd_capi.cu (thread-local kd_last_error message)
int kd_set_error(int code, const char* msg);

namespace {
struct Buf {
    void* p = nullptr;
    cudaStream_t st;
    Buf(size_t b, cudaStream_t s) : st(s) { KD_CUDA(cudaMallocAsync(&p, b ? b : 1, s)); }
    ~Buf() {
        if (p) cudaFreeAsync(p, st);
    }
};
int derr(int code, const std::string& m) { return kd_set_error(code, m.c_str()); }
}  // namespace

#define KD_DTRY(...)                                                   \
    try {                                                              \
        __VA_ARGS__;                                                   \
    } catch (const kdb::CudaError& e) {                                \
        return derr(KD_ECUDA, e.msg);                                  \
    } catch (const std::exception& e) {                                \
        return derr(KD_ECUDA, e.what());                               \
    }

extern "C" {

KD_API int kd_histogram(const void* values, int dtype, int64_t n, const double* boundaries, int64_t nb,
                        int64_t* counts, int64_t* equals, unsigned flags, void* stream) {
    if (nb < 1 || nb > HIST_MAXB) return derr(KD_EUNSUPPORTED, "kd_histogram: nb must be in [1, 4096]");
    if (n < 0) return derr(KD_EINVAL, "kd_histogram: n < 0");
    if (dtype != KD_F32 && dtype != KD_F64) return derr(KD_EINVAL, "kd_histogram: bad dtype");
    KD_DTRY({
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const bool dp = flags & KD_DEVICE_PTRS;
        const size_t es = dtype == KD_F32 ? 4 : 8;
        Buf dv(dp ? 0 : n * es, st), db(dp ? 0 : nb * 8, st), dc((nb + 1) * 8, st), de(nb * 8, st);
        const void* v = values;
        const double* b = boundaries;
        if (!dp) {
            if (n) KD_CUDA(cudaMemcpyAsync(dv.p, values, n * es, cudaMemcpyHostToDevice, st));
            KD_CUDA(cudaMemcpyAsync(db.p, boundaries, nb * 8, cudaMemcpyHostToDevice, st));
            v = dv.p;
            b = (const double*)db.p;
        }
        KD_CUDA(cudaMemsetAsync(dc.p, 0, (nb + 1) * 8, st));
        KD_CUDA(cudaMemsetAsync(de.p, 0, nb * 8, st));
        if (n) {
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const unsigned grid = (unsigned)std::min<int64_t>((n + HIST_THREADS - 1) / HIST_THREADS, (int64_t)sms * 4);
            const size_t sm = (size_t)nb * 8 + (size_t)(nb + 1) * 4 + (size_t)nb * 4;
            KD_CUDA(cudaFuncSetAttribute(k_hist_full<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000));
            KD_CUDA(cudaFuncSetAttribute(k_hist_full<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000));
            if (dtype == KD_F32)
                k_hist_full<float><<<grid, HIST_THREADS, sm, st>>>((const float*)v, n, b, (int)nb,
                                                                 (unsigned long long*)dc.p, (unsigned long long*)de.p);
            else
                k_hist_full<double><<<grid, HIST_THREADS, sm, st>>>((const double*)v, n, b, (int)nb,
                                                                  (unsigned long long*)dc.p, (unsigned long long*)de.p);
            KD_CUDA(cudaGetLastError());
        }
        const cudaMemcpyKind kind = dp ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        KD_CUDA(cudaMemcpyAsync(counts, dc.p, (nb + 1) * 8, kind, st));
        if (equals) KD_CUDA(cudaMemcpyAsync(equals, de.p, nb * 8, kind, st));
        KD_CUDA(cudaStreamSynchronize(st));
    });
    return KD_OK;
}

KD_API int kd_partition(const void* coords, int dtype, int64_t n, int dims, const uint64_t* ids, int dim,
                        double value, void* out_coords, uint64_t* out_ids, int64_t* n_low, unsigned flags,
                        void* stream) {
    if (!(flags & KD_DEVICE_PTRS)) return derr(KD_EINVAL, "kd_partition: device pointers required");
    if (dim < 0 || dim >= dims) return derr(KD_EINVAL, "kd_partition: dim out of range");
    if (dtype != KD_F32 && dtype != KD_F64) return derr(KD_EINVAL, "kd_partition: bad dtype");
    if (!n_low) return derr(KD_EINVAL, "kd_partition: n_low is NULL");
    if (n == 0) { *n_low = 0; return KD_OK; }
    KD_DTRY({
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        Buf fl(n * 4, st), pre(n * 8, st), tot(8, st);
        const unsigned g = (unsigned)((n + 255) / 256);
        const size_t es = dtype == KD_F32 ? 4 : 8;
        const char* row = static_cast<const char*>(coords) + (size_t)dim * n * es;
        if (dtype == KD_F32) k_flag_low<float><<<g, 256, 0, st>>>((const float*)row, n, value, (int32_t*)fl.p);
        else k_flag_low<double><<<g, 256, 0, st>>>((const double*)row, n, value, (int32_t*)fl.p);
        size_t tb = 0;
        cub::TransformInputIterator<int64_t, cub::CastOp<int64_t>, const int32_t*> it((const int32_t*)fl.p,
                                                                                     cub::CastOp<int64_t>());
        cub::DeviceScan::ExclusiveSum(nullptr, tb, it, (int64_t*)pre.p, (int)n, st);
        Buf tmp(tb, st);
        cub::DeviceScan::ExclusiveSum(tmp.p, tb, it, (int64_t*)pre.p, (int)n, st);
        int64_t last_pre = 0;
        int32_t last_flag = 0;
        KD_CUDA(cudaMemcpyAsync(&last_pre, (int64_t*)pre.p + n - 1, 8, cudaMemcpyDeviceToHost, st));
        KD_CUDA(cudaMemcpyAsync(&last_flag, (int32_t*)fl.p + n - 1, 4, cudaMemcpyDeviceToHost, st));
        KD_CUDA(cudaStreamSynchronize(st));
        const int64_t nl = last_pre + last_flag;
        if (dtype == KD_F32)
            k_part_scatter<float><<<g, 256, 0, st>>>((const float*)coords, ids, n, dims, (int32_t*)fl.p,
                                                     (int64_t*)pre.p, nl, (float*)out_coords, out_ids);
        else
            k_part_scatter<double><<<g, 256, 0, st>>>((const double*)coords, ids, n, dims, (int32_t*)fl.p,
                                                      (int64_t*)pre.p, nl, (double*)out_coords, out_ids);
        KD_CUDA(cudaGetLastError());
        KD_CUDA(cudaStreamSynchronize(st));
        *n_low = nl;
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

}  // extern "C"
