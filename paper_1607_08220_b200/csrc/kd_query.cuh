// kd_query.cuh -- exact KNN entry point (device pointers only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kd_tree.cuh"

namespace kdb {

struct KnnArgs {
    const double* queries = nullptr;  // [nq][dims] row-major binary64
    int64_t nq = 0;
    int64_t k = 1;
    const double* radii = nullptr;    // [nq] squared radii (nullptr = +inf)
    const uint64_t* excl = nullptr;   // [nq] id to exclude per query (nullptr = none)
    double* out_d = nullptr;          // [nq][k]
    uint64_t* out_i = nullptr;        // [nq][k]
    int64_t* out_c = nullptr;         // [nq]
    int64_t* out_ctr = nullptr;       // [nq][3] or nullptr
    double* heap_d = nullptr;         // [nq][k] scratch when k > 32
    uint64_t* heap_i = nullptr;
    bool sort_queries = true;
    bool thread_per_query = false;  // one-thread-per-query traversal (k > 32 always uses it)
    bool packet = false;            // D <= 3: warp-per-packet kernel (kd_packet.cu) instead of per-lane traversals
};

constexpr int KNN_MAX_DEPTH = 37;  // traversal stack capacity - 3
constexpr int64_t KNN_CHUNK_MIN = 1 << 20;  // host-buffer pipeline: queries per chunk (at least)
constexpr int64_t KNN_MAX_CHUNKS = 16;

void knn(const KdTreeDev& t, const KnnArgs& a, cudaStream_t st);
// kd_walk.cu: any depth / any k; reference = true walks exactly as local_query.py:72-172 (results and counters)
void knn_walk(const KdTreeDev& t, const KnnArgs& a, bool reference, cudaStream_t st);
bool knn_packet(const KdTreeDev& t, const KnnArgs& a, const int32_t* order, cudaStream_t st);  // kd_packet.cu

}  // namespace kdb
