// kd_tree.cuh -- device-resident kd-tree layout shared by build, query and the C-ABI.
//
// Nodes are stored in the reference's canonical preorder (local_tree.py:320-374),
// so the left child of interior node i is i+1.  One 16-byte record per node:
//   interior: v = split value (binary64), a = right child, db = split dim (>= 0)
//   leaf    : a = first packed row, db = -1 - bucket length
// Packed points are SoA [dims][n] of the storage type (float or double);
// ids are the caller's uint64 ids in packed order.
#pragma once
#include <stdint.h>

namespace kdb {

struct __align__(16) KdNode {
    double v;
    int32_t a;
    int32_t db;
};

// query-tree record for D <= 3 (kd_packet.cu): one per interior node, holding
// both children's tight f32 bounding boxes (lo[0..2], hi[0..2]) and references
// -- an interior child node index (count < 0) or a leaf bucket [ref, ref + count)
struct __align__(16) QNode {
    float lb[6];
    float rb[6];
    int32_t l, lc, r, rc;
};

enum { DT_F32 = 1, DT_F64 = 2 };

struct KdTreeDev {
    int device = 0;
    int dims = 0;
    int dtype = DT_F32;
    int64_t n = 0;
    int64_t n_nodes = 0;
    int64_t n_leaves = 0;
    int64_t depth = 0;
    KdNode* nodes = nullptr;     // [n_nodes]
    int32_t* node_count = nullptr;  // [n_nodes] points under each node
    void* coords = nullptr;      // [dims][n] packed, float or double
    uint64_t* ids = nullptr;     // [n] packed ids
    int32_t* perm = nullptr;     // [n] packed row i holds input row perm[i]
    QNode* qnodes = nullptr;     // [n_nodes] query tree (D <= 3; built with the tree)
};

struct BuildCfg {
    int64_t bucket = 32;
    int64_t msample = 1024;   // local_sample_m
    int64_t vsample = 1024;   // variance_sample
    uint64_t seed = 0;
};

struct BuildStats {
    double ms_total = 0;
    double ms_levels = 0, ms_subtree = 0, ms_finish = 0;  // phase split of ms_total
    int levels = 0;        // breadth-first (global-memory) levels
    int64_t tasks = 0;     // shared-memory subtree tasks
    int64_t slow_nodes = 0;  // nodes that needed the exact slow path
};

template <typename T>
void build_tree(const T* d_coords_soa, const uint64_t* d_ids, int64_t n, int dims, const BuildCfg& cfg,
                cudaStream_t st, KdTreeDev* out, BuildStats* stats);

void free_tree(KdTreeDev* t);
void build_qtree(KdTreeDev* t, cudaStream_t st);  // kd_packet.cu
void retain_pool(int device);

}  // namespace kdb
