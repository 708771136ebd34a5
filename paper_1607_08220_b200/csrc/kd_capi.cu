// kd_capi.cu -- extern "C" boundary (include/kdtree_b200.h) over the device build/query.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <new>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/kdtree_b200.h"
#include "kd_common.cuh"
#include "kd_arena.cuh"
#include "kd_query.cuh"
#include "kd_tree.cuh"

using namespace kdb;

struct kd_tree {
    KdTreeDev dev;
    BuildStats stats;
    std::mutex mu;  // guards the lazily built query tree
};

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

int kd_set_error(int code, const char* msg) { return fail(code, msg); }

#define KD_TRY(...)                                                                    \
    try {                                                                              \
        __VA_ARGS__;                                                                        \
    } catch (const kdb::CudaError& e) {                                                \
        return fail(KD_ECUDA, e.msg);                                                  \
    } catch (const std::bad_alloc&) {                                                  \
        return fail(KD_ENOMEM, "host allocation failed");                              \
    } catch (const std::exception& e) {                                                \
        return fail(KD_ECUDA, e.what());                                               \
    }

namespace {

// scratch for one call: from the calling thread's arena inside an ArenaScope (synchronous
// host-buffer paths), else from the stream-ordered pool
struct DevBuf {
    void* p = nullptr;
    cudaStream_t st = nullptr;
    bool arena = false;
    DevBuf() = default;
    DevBuf(size_t bytes, cudaStream_t s) : st(s) {
        if (t_arena) {
            p = t_arena->alloc(bytes);
            arena = true;
        } else {
            KD_CUDA(cudaMallocAsync(&p, bytes ? bytes : 1, s));
        }
    }
    ~DevBuf() {
        if (p && !arena) cudaFreeAsync(p, st);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        KD_CUDA(cudaGetDevice(&prev));
        if (prev != dev) KD_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

__global__ void k_export(const KdNode* nodes, const int32_t* ncount, int64_t nn, int32_t* dim, double* val,
                         int32_t* left, int32_t* right, int64_t* cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
    const KdNode r = nodes[i];
    if (r.db >= 0) {
        dim[i] = r.db; val[i] = r.v; left[i] = (int32_t)(i + 1); right[i] = r.a;
    } else {
        dim[i] = -1; val[i] = 0.0; left[i] = r.a; right[i] = -1 - r.db;
    }
    cnt[i] = ncount[i];
}

template <typename T>
__global__ void k_coords_f64(const T* in, double* out, int64_t count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) out[i] = (double)in[i];
}

__global__ void k_import(const int32_t* dim, const double* val, const int32_t* left, const int32_t* right,
                         const int64_t* cnt, int64_t nn, KdNode* nodes, int32_t* ncount, int* bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= nn) return;
    if (dim[i] >= 0) {
        if (left[i] != i + 1) atomicExch(bad, 1);  // not in preorder
        nodes[i] = KdNode{val[i], right[i], dim[i]};
    } else {
        nodes[i] = KdNode{0.0, left[i], -1 - right[i]};
    }
    ncount[i] = (int32_t)cnt[i];
}

__global__ void k_f64_to_f32(const double* in, float* out, int64_t count) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) out[i] = (float)in[i];
}

}  // namespace

extern "C" {

int kd_version(void) { return 10000; }

const char* kd_last_error(void) { return g_err.c_str(); }

int kd_device_count(int* count) {
    if (!count) return fail(KD_EINVAL, "count is NULL");
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(KD_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    return KD_OK;
}

int kd_tree_build(const void* coords, int dtype, int64_t n, int dims, const uint64_t* ids, const kd_build_cfg* cfg,
                  int device, unsigned flags, void* stream, kd_tree** out) {
    if (!out) return fail(KD_EINVAL, "out is NULL");
    *out = nullptr;
    if (dims < 1 || dims > 16) return fail(KD_EUNSUPPORTED, "dims must be in [1, 16] on the device");
    if (n < 0 || n >= (int64_t(1) << 30)) return fail(KD_EUNSUPPORTED, "n must be in [0, 2^30) per device");
    if (dtype != KD_F32 && dtype != KD_F64) return fail(KD_EINVAL, "dtype must be KD_F32 or KD_F64");
    if (n > 0 && !coords) return fail(KD_EINVAL, "coords is NULL");
    BuildCfg bc;
    if (cfg) {
        bc.bucket = cfg->bucket_size;
        bc.msample = cfg->local_sample_m;
        bc.vsample = cfg->variance_sample;
        bc.seed = cfg->seed;
    }
    if (bc.bucket < 1) return fail(KD_EINVAL, "bucket_size must be >= 1");
    if (bc.msample < 1 || bc.vsample < 1) return fail(KD_EINVAL, "sample sizes must be >= 1");
    if (bc.msample > 1024 || bc.vsample > 1024)
        return fail(KD_EUNSUPPORTED, "sample sizes above 1024 are not supported on the device");
    KD_TRY({
        DeviceGuard g(device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const size_t es = dtype == KD_F32 ? 4 : 8;
        const bool dev_ptrs = flags & KD_DEVICE_PTRS;
        DevBuf hc, hi;
        const void* dc = coords;
        const uint64_t* di = ids;
        std::unique_ptr<ArenaScope> scope;
        if (!dev_ptrs && n > 0) scope.reset(new ArenaScope(device));  // staging lives until the build returns
        if (!dev_ptrs && n > 0) {
            hc.~DevBuf();
            new (&hc) DevBuf((size_t)dims * n * es, st);
            KD_CUDA(cudaMemcpyAsync(hc.p, coords, (size_t)dims * n * es, cudaMemcpyHostToDevice, st));
            dc = hc.p;
            if (ids) {
                new (&hi) DevBuf((size_t)n * 8, st);
                KD_CUDA(cudaMemcpyAsync(hi.p, ids, (size_t)n * 8, cudaMemcpyHostToDevice, st));
                di = static_cast<const uint64_t*>(hi.p);
            }
        }
        kd_tree* t = new kd_tree();
        try {
            if (dtype == KD_F32)
                build_tree<float>(static_cast<const float*>(dc), di, n, dims, bc, st, &t->dev, &t->stats);
            else
                build_tree<double>(static_cast<const double*>(dc), di, n, dims, bc, st, &t->dev, &t->stats);
        } catch (...) {
            free_tree(&t->dev);
            delete t;
            throw;
        }
        *out = t;
    });
    return KD_OK;
}

int kd_tree_import(const kd_tree_arrays* a, int64_t n_nodes, int64_t n, int dims, int64_t depth, int dtype,
                   int device, kd_tree** out) {
    if (!a || !out) return fail(KD_EINVAL, "NULL argument");
    *out = nullptr;
    if (dims < 1 || dims > 16) return fail(KD_EUNSUPPORTED, "dims must be in [1, 16] on the device");
    if (n_nodes < 0 || n < 0) return fail(KD_EINVAL, "negative size");
    if (dtype != KD_F32 && dtype != KD_F64) return fail(KD_EINVAL, "dtype must be KD_F32 or KD_F64");
    KD_TRY({
        DeviceGuard g(device);
        cudaStream_t st = 0;
        kd_tree* t = new kd_tree();
        KdTreeDev& d = t->dev;
        d.device = device; d.dims = dims; d.dtype = dtype; d.n = n; d.n_nodes = n_nodes; d.depth = depth;
        const int64_t nn1 = n_nodes > 0 ? n_nodes : 1, n1 = n > 0 ? n : 1;
        retain_pool(device);
        KD_CUDA(cudaMallocAsync((void**)&d.nodes, nn1 * sizeof(KdNode), st));
        KD_CUDA(cudaMallocAsync((void**)&d.node_count, nn1 * sizeof(int32_t), st));
        KD_CUDA(cudaMallocAsync((void**)&d.ids, n1 * 8, st));
        KD_CUDA(cudaMallocAsync((void**)&d.perm, n1 * 4, st));
        KD_CUDA(cudaMallocAsync(&d.coords, (size_t)dims * n1 * (dtype == KD_F32 ? 4 : 8), st));
        if (n_nodes > 0) {
            DevBuf bdim(nn1 * 4, st), bval(nn1 * 8, st), bl(nn1 * 4, st), br(nn1 * 4, st), bc(nn1 * 8, st), bad(4, st);
            KD_CUDA(cudaMemcpyAsync(bdim.p, a->node_dim, n_nodes * 4, cudaMemcpyHostToDevice, st));
            KD_CUDA(cudaMemcpyAsync(bval.p, a->node_value, n_nodes * 8, cudaMemcpyHostToDevice, st));
            KD_CUDA(cudaMemcpyAsync(bl.p, a->node_left, n_nodes * 4, cudaMemcpyHostToDevice, st));
            KD_CUDA(cudaMemcpyAsync(br.p, a->node_right, n_nodes * 4, cudaMemcpyHostToDevice, st));
            KD_CUDA(cudaMemcpyAsync(bc.p, a->node_count, n_nodes * 8, cudaMemcpyHostToDevice, st));
            KD_CUDA(cudaMemsetAsync(bad.p, 0, 4, st));
            k_import<<<(unsigned)((n_nodes + 255) / 256), 256, 0, st>>>(
                (int32_t*)bdim.p, (double*)bval.p, (int32_t*)bl.p, (int32_t*)br.p, (int64_t*)bc.p, n_nodes, d.nodes,
                d.node_count, (int*)bad.p);
            int hbad = 0;
            KD_CUDA(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, st));
            KD_CUDA(cudaStreamSynchronize(st));
            if (hbad) {
                free_tree(&d);
                delete t;
                return fail(KD_EINVAL, "imported tree is not in preorder (left child != node + 1)");
            }
            int64_t leaves = 0;
            for (int64_t i = 0; i < n_nodes; i++) leaves += a->node_dim[i] < 0;
            d.n_leaves = leaves;
        }
        if (n > 0) {
            KD_CUDA(cudaMemcpyAsync(d.ids, a->ids, n * 8, cudaMemcpyHostToDevice, st));
            if (dtype == KD_F64) {
                KD_CUDA(cudaMemcpyAsync(d.coords, a->coords, (size_t)dims * n * 8, cudaMemcpyHostToDevice, st));
            } else {
                DevBuf tmp((size_t)dims * n * 8, st);
                KD_CUDA(cudaMemcpyAsync(tmp.p, a->coords, (size_t)dims * n * 8, cudaMemcpyHostToDevice, st));
                k_f64_to_f32<<<(unsigned)(((int64_t)dims * n + 255) / 256), 256, 0, st>>>(
                    (double*)tmp.p, (float*)d.coords, (int64_t)dims * n);
            }
            std::vector<int32_t> iota(n);
            for (int64_t i = 0; i < n; i++) iota[i] = (int32_t)i;
            KD_CUDA(cudaMemcpyAsync(d.perm, iota.data(), n * 4, cudaMemcpyHostToDevice, st));
        }
        KD_CUDA(cudaStreamSynchronize(st));
        *out = t;
    });
    return KD_OK;
}

int kd_tree_get_info(const kd_tree* t, kd_tree_info* info) {
    if (!t || !info) return fail(KD_EINVAL, "NULL argument");
    std::memset(info, 0, sizeof(*info));
    info->n_nodes = t->dev.n_nodes;
    info->n = t->dev.n;
    info->n_leaves = t->dev.n_leaves;
    info->depth = t->dev.depth;
    info->dims = t->dev.dims;
    info->dtype = t->dev.dtype;
    info->device = t->dev.device;
    info->build_ms = t->stats.ms_total;
    info->build_ms_levels = t->stats.ms_levels;
    info->build_ms_subtree = t->stats.ms_subtree;
    info->build_ms_finish = t->stats.ms_finish;
    info->build_levels = t->stats.levels;
    info->build_tasks = t->stats.tasks;
    info->build_slow_nodes = t->stats.slow_nodes;
    return KD_OK;
}

int kd_tree_export(const kd_tree* t, kd_tree_arrays* o) {
    if (!t || !o) return fail(KD_EINVAL, "NULL argument");
    KD_TRY({
        const KdTreeDev& d = t->dev;
        DeviceGuard g(d.device);
        cudaStream_t st = 0;
        const int64_t nn = d.n_nodes, n = d.n;
        if (nn > 0) {
            DevBuf bdim(nn * 4, st), bval(nn * 8, st), bl(nn * 4, st), br(nn * 4, st), bc(nn * 8, st);
            k_export<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(d.nodes, d.node_count, nn, (int32_t*)bdim.p,
                                                                  (double*)bval.p, (int32_t*)bl.p, (int32_t*)br.p,
                                                                  (int64_t*)bc.p);
            KD_CUDA(cudaGetLastError());
            if (o->node_dim) KD_CUDA(cudaMemcpyAsync(o->node_dim, bdim.p, nn * 4, cudaMemcpyDeviceToHost, st));
            if (o->node_value) KD_CUDA(cudaMemcpyAsync(o->node_value, bval.p, nn * 8, cudaMemcpyDeviceToHost, st));
            if (o->node_left) KD_CUDA(cudaMemcpyAsync(o->node_left, bl.p, nn * 4, cudaMemcpyDeviceToHost, st));
            if (o->node_right) KD_CUDA(cudaMemcpyAsync(o->node_right, br.p, nn * 4, cudaMemcpyDeviceToHost, st));
            if (o->node_count) KD_CUDA(cudaMemcpyAsync(o->node_count, bc.p, nn * 8, cudaMemcpyDeviceToHost, st));
            KD_CUDA(cudaStreamSynchronize(st));
        }
        if (n > 0) {
            if (o->coords) {
                const int64_t cnt = (int64_t)d.dims * n;
                if (d.dtype == KD_F64) {
                    KD_CUDA(cudaMemcpyAsync(o->coords, d.coords, cnt * 8, cudaMemcpyDeviceToHost, st));
                } else {
                    DevBuf tmp(cnt * 8, st);
                    k_coords_f64<float><<<(unsigned)((cnt + 255) / 256), 256, 0, st>>>((const float*)d.coords,
                                                                                      (double*)tmp.p, cnt);
                    KD_CUDA(cudaMemcpyAsync(o->coords, tmp.p, cnt * 8, cudaMemcpyDeviceToHost, st));
                    KD_CUDA(cudaStreamSynchronize(st));
                }
            }
            if (o->ids) KD_CUDA(cudaMemcpyAsync(o->ids, d.ids, n * 8, cudaMemcpyDeviceToHost, st));
            if (o->perm) {
                std::vector<int32_t> p32(n);
                KD_CUDA(cudaMemcpyAsync(p32.data(), d.perm, n * 4, cudaMemcpyDeviceToHost, st));
                KD_CUDA(cudaStreamSynchronize(st));
                for (int64_t i = 0; i < n; i++) o->perm[i] = p32[i];
            }
            KD_CUDA(cudaStreamSynchronize(st));
        }
    });
    return KD_OK;
}

int kd_knn(const kd_tree* t, const double* queries, int64_t nq, int64_t k, const double* radii,
           const uint64_t* exclude_ids, double* out_d, uint64_t* out_i, int64_t* out_c, int64_t* out_ctr,
           unsigned flags, void* stream) {
    if (!t) return fail(KD_EINVAL, "tree is NULL");
    if (k < 1) return fail(KD_EINVAL, "k must be >= 1");
    if (nq < 0) return fail(KD_EINVAL, "nq must be >= 0");
    if (nq >= (int64_t(1) << 31)) return fail(KD_EUNSUPPORTED, "nq must be < 2^31 per call");
    if (nq > 0 && (!queries || !out_d || !out_i || !out_c)) return fail(KD_EINVAL, "NULL query/output buffer");
    // the packet kernel (D <= 3, k(+1) <= 32) sizes its stack from the tree depth; the
    // per-query kernels carry a fixed stack
    const bool packet = (flags & KD_KNN_PACKET) && t->dev.dims <= 3 && k + (exclude_ids ? 1 : 0) <= 32 &&
                        !(flags & KD_THREAD_PER_QUERY);
    const bool ref_walk = (flags & KD_KNN_REFERENCE) != 0;
    if (ref_walk && exclude_ids) return fail(KD_EINVAL, "KD_KNN_REFERENCE: the reference walk has no id exclusion");
    // trees deeper than the fast kernels' fixed stack take the depth-sized walk (kd_walk.cu)
    const bool walk = ref_walk || (!packet && t->dev.depth > KNN_MAX_DEPTH);
    if (nq == 0) return KD_OK;
    KD_TRY({
        const KdTreeDev& d = t->dev;
        DeviceGuard g(d.device);
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        const bool dev_ptrs = flags & KD_DEVICE_PTRS;
        const int D = d.dims;
        KnnArgs a;
        a.nq = nq;
        a.k = k;
        a.sort_queries = !(flags & KD_NO_SORT);
        a.thread_per_query = (flags & KD_THREAD_PER_QUERY) != 0;
        a.packet = (flags & KD_KNN_PACKET) != 0;
        if (a.packet && !walk) {  // the packet kernel's query tree (tight boxes) is built on first use
            std::lock_guard<std::mutex> lk(const_cast<kd_tree*>(t)->mu);
            if (!d.qnodes) build_qtree(const_cast<KdTreeDev*>(&d), st);
        }
        DevBuf bq, br, be, bd, bi, bc, bctr;
        DevBuf hd, hi;
        if (!walk && (k > 32 || (k == 32 && exclude_ids && !a.thread_per_query))) {  // heap kernel scratch
            new (&hd) DevBuf(nq * k * 8, st);
            new (&hi) DevBuf(nq * k * 8, st);
            a.heap_d = (double*)hd.p;
            a.heap_i = (uint64_t*)hi.p;
        }
        if (dev_ptrs) {
            a.queries = queries; a.radii = radii; a.excl = exclude_ids;
            a.out_d = out_d; a.out_i = out_i; a.out_c = out_c; a.out_ctr = out_ctr;
            if (walk) knn_walk(d, a, ref_walk, st);
            else knn(d, a, st);
            return KD_OK;
        }
        ArenaScope scope(d.device);  // synchronous below: staging from the arena
        // host buffers: device staging for the whole batch, then a pipeline over
        // query chunks -- H2D of chunk c+1 and D2H of chunk c-1 (copy engines, one
        // per direction) overlap the search of chunk c on the caller's stream
        new (&bq) DevBuf(nq * D * 8, st);
        if (radii) new (&br) DevBuf(nq * 8, st);
        if (exclude_ids) new (&be) DevBuf(nq * 8, st);
        new (&bd) DevBuf(nq * k * 8, st);
        new (&bi) DevBuf(nq * k * 8, st);
        new (&bc) DevBuf(nq * 8, st);
        if (out_ctr) new (&bctr) DevBuf(nq * 3 * 8, st);
        static const int64_t max_chunks = [] {  // KDB_KNN_CHUNKS overrides (A/B measurements)
            const char* e = std::getenv("KDB_KNN_CHUNKS");
            return e ? std::max<int64_t>(1, atoll(e)) : KNN_MAX_CHUNKS;
        }();
        const int64_t nch = std::max<int64_t>(1, std::min<int64_t>(max_chunks, nq / KNN_CHUNK_MIN));
        const int64_t csz = (nq + nch - 1) / nch;
        // copy streams + events; on every exit path (incl. a throw mid-pipeline) the guard waits
        // for both copy streams and the caller's stream before the staging buffers go away
        struct Pipe {
            cudaStream_t s_in = nullptr, s_out = nullptr, st = nullptr;
            std::vector<cudaEvent_t> evs;
            ~Pipe() {
                if (s_in) cudaStreamSynchronize(s_in);
                if (s_out) cudaStreamSynchronize(s_out);
                if (st) cudaStreamSynchronize(st);
                for (auto& e : evs)
                    if (e) cudaEventDestroy(e);
                if (s_in) cudaStreamDestroy(s_in);
                if (s_out) cudaStreamDestroy(s_out);
            }
        } pipe;
        pipe.st = st;
        KD_CUDA(cudaStreamCreateWithFlags(&pipe.s_in, cudaStreamNonBlocking));
        KD_CUDA(cudaStreamCreateWithFlags(&pipe.s_out, cudaStreamNonBlocking));
        cudaStream_t s_in = pipe.s_in, s_out = pipe.s_out;
        pipe.evs.assign(2 * nch + 2, nullptr);
        std::vector<cudaEvent_t>& evs = pipe.evs;
        for (auto& e : evs) KD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        KD_CUDA(cudaEventRecord(evs[2 * nch], st));  // staging allocated
        KD_CUDA(cudaStreamWaitEvent(s_in, evs[2 * nch], 0));
        KD_CUDA(cudaStreamWaitEvent(s_out, evs[2 * nch], 0));
        for (int64_t c = 0; c < nch; c++) {
            const int64_t lo = c * csz, cnt = std::min(csz, nq - lo);
            if (cnt <= 0) break;
            KD_CUDA(cudaMemcpyAsync((double*)bq.p + lo * D, queries + lo * D, cnt * D * 8, cudaMemcpyHostToDevice, s_in));
            if (radii) KD_CUDA(cudaMemcpyAsync((double*)br.p + lo, radii + lo, cnt * 8, cudaMemcpyHostToDevice, s_in));
            if (exclude_ids)
                KD_CUDA(cudaMemcpyAsync((uint64_t*)be.p + lo, exclude_ids + lo, cnt * 8, cudaMemcpyHostToDevice, s_in));
            KD_CUDA(cudaEventRecord(evs[2 * c], s_in));
            KD_CUDA(cudaStreamWaitEvent(st, evs[2 * c], 0));
            KnnArgs ac = a;
            ac.nq = cnt;
            ac.queries = (const double*)bq.p + lo * D;
            ac.radii = radii ? (const double*)br.p + lo : nullptr;
            ac.excl = exclude_ids ? (const uint64_t*)be.p + lo : nullptr;
            ac.out_d = (double*)bd.p + lo * k;
            ac.out_i = (uint64_t*)bi.p + lo * k;
            ac.out_c = (int64_t*)bc.p + lo;
            ac.out_ctr = out_ctr ? (int64_t*)bctr.p + lo * 3 : nullptr;
            if (a.heap_d) { ac.heap_d = a.heap_d + lo * k; ac.heap_i = a.heap_i + lo * k; }
            if (walk) knn_walk(d, ac, ref_walk, st);
            else knn(d, ac, st);
            KD_CUDA(cudaEventRecord(evs[2 * c + 1], st));
            KD_CUDA(cudaStreamWaitEvent(s_out, evs[2 * c + 1], 0));
            KD_CUDA(cudaMemcpyAsync(out_d + lo * k, ac.out_d, cnt * k * 8, cudaMemcpyDeviceToHost, s_out));
            KD_CUDA(cudaMemcpyAsync(out_i + lo * k, ac.out_i, cnt * k * 8, cudaMemcpyDeviceToHost, s_out));
            KD_CUDA(cudaMemcpyAsync(out_c + lo, ac.out_c, cnt * 8, cudaMemcpyDeviceToHost, s_out));
            if (out_ctr) KD_CUDA(cudaMemcpyAsync(out_ctr + lo * 3, ac.out_ctr, cnt * 3 * 8, cudaMemcpyDeviceToHost, s_out));
        }
        // the caller's stream (and the staging frees queued on it) follows the last copy-out
        KD_CUDA(cudaEventRecord(evs[2 * nch + 1], s_out));
        KD_CUDA(cudaStreamWaitEvent(st, evs[2 * nch + 1], 0));
        KD_CUDA(cudaStreamSynchronize(s_out));
        KD_CUDA(cudaStreamSynchronize(st));
    });
    return KD_OK;
}

int kd_tree_free(kd_tree* t) {
    if (!t) return KD_OK;
    int cur = -1;
    cudaGetDevice(&cur);
    cudaSetDevice(t->dev.device);
    cudaDeviceSynchronize();
    free_tree(&t->dev);
    if (cur >= 0) cudaSetDevice(cur);
    delete t;
    return KD_OK;
}

}  // extern "C"
