// kd_arena.cuh -- per-device scratch arenas (chunked bump allocators reused across calls).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <vector>

#include "kd_common.cuh"

namespace kdb {

// Build scratch comes from a per-device arena of persistent chunks reused by every
// build (bump allocation, reset per build): the stream-ordered pool stalled for
// 10-400 ms on some of a 256M-point build's ~100 allocations (growth/remapping of a
// fragmented pool), while a build's allocation sequence is the same from one build to
// the next, so the chunks fit again without touching the driver.  Only the buffers
// the tree keeps (packed coordinates, row ids, ids, nodes, counts) use the pool.
struct Arena {
    int device = 0;
    struct Chunk {
        char* base;
        size_t size;
    };
    std::vector<Chunk> chunks;
    size_t ci = 0, off = 0;
    void reset() { ci = 0; off = 0; }
    bool owns(const void* p) const {
        for (const Chunk& c : chunks)
            if ((const char*)p >= c.base && (const char*)p < c.base + c.size) return true;
        return false;
    }
    void* alloc(size_t bytes) {
        bytes = (std::max<size_t>(bytes, 1) + 255) & ~(size_t)255;
        while (ci < chunks.size()) {
            if (off + bytes <= chunks[ci].size) {
                void* p = chunks[ci].base + off;
                off += bytes;
                return p;
            }
            ci++;
            off = 0;
        }
        const size_t sz = std::max<size_t>(bytes, (size_t)1 << 28);
        char* p = nullptr;
        KD_CUDA(cudaMalloc(&p, sz));  // growth only (first build of a size)
        chunks.push_back({p, sz});
        off = bytes;
        return p;
    }
};
Arena* arena_acquire(int device);  // kd_build_f32.cu (one free list per device)
void arena_release(Arena* a);
inline thread_local Arena* t_arena = nullptr;

struct ArenaScope {  // the calling thread's scratch comes from `a` while in scope (synchronous callers)
    Arena* a;
    Arena* prev;
    explicit ArenaScope(int device) : a(arena_acquire(device)), prev(t_arena) { t_arena = a; }
    ~ArenaScope() {
        t_arena = prev;
        arena_release(a);
    }
};


// An arena bound to a (device, stream): calls that enqueue asynchronous work take their
// temporaries from it; the next call on the same stream reuses it in stream order (the
// earlier kernels finish before the later ones start), so no allocation and no sync.
struct StreamArena {
    std::unique_lock<std::mutex> lk;
    Arena* prev;
    StreamArena(int dev, cudaStream_t s) {
        static std::mutex mu;
        static std::map<std::pair<int, cudaStream_t>, std::pair<Arena*, std::mutex*>> by_stream;
        std::pair<Arena*, std::mutex*> e;
        {
            std::lock_guard<std::mutex> g(mu);
            auto it = by_stream.find({dev, s});
            if (it == by_stream.end()) {
                Arena* a = new Arena();
                a->device = dev;
                it = by_stream.emplace(std::make_pair(dev, s), std::make_pair(a, new std::mutex())).first;
            }
            e = it->second;
        }
        lk = std::unique_lock<std::mutex>(*e.second);  // one host thread enqueues on a stream at a time
        e.first->reset();
        prev = t_arena;
        t_arena = e.first;
    }
    ~StreamArena() { t_arena = prev; }
    StreamArena(const StreamArena&) = delete;
    StreamArena& operator=(const StreamArena&) = delete;
};

template <typename X>
inline X* scratch(size_t count, cudaStream_t st) {
    if (t_arena) return static_cast<X*>(t_arena->alloc(std::max<size_t>(count, 1) * sizeof(X)));
    void* p = nullptr;
    KD_CUDA(cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(X), st));
    return static_cast<X*>(p);
}
inline void scratch_free(void* p, cudaStream_t st) {
    if (p && !(t_arena && t_arena->owns(p))) cudaFreeAsync(p, st);
}

}  // namespace kdb
