// memory.cu -- device scratch allocation (see common.cuh: Buf).
//
// Large blocks are cached here instead of being returned to the stream-
// ordered pool: re-mapping physical pages for a fresh multi-GB range costs
// ~6 ms per GB on B200, more than the contraction that needs the buffer.
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.cuh"

namespace lcc {
namespace {

struct Block {
    void* p;
    size_t cap;
    cudaStream_t s;
    cudaEvent_t ready;  // recorded on s at release: reuse on another stream waits on it
};

struct Cache {
    std::mutex m;
    std::multimap<size_t, Block> free;  // by capacity
    size_t held = 0;                    // bytes in `free`
};

Cache& cache() {
    static Cache c[16];
    int dev = 0;
    cudaGetDevice(&dev);
    return c[dev & 15];
}

constexpr size_t GRAIN = 2ull << 20;

// diagnostics: LCC_ALLOC_FILL=<byte> fills every fresh scratch block, so a
// kernel that reads memory it never wrote shows up in every run
int alloc_fill() {
    static const int f = getenv("LCC_ALLOC_FILL") ? (int)strtol(getenv("LCC_ALLOC_FILL"), nullptr, 0) : -1;
    return f;
}

}  // namespace

void* pool_alloc(size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e == cudaErrorMemoryAllocation) {
        // First hand the library's cached blocks back to the pool: the pool
        // keeps that memory mapped and can serve the request from it (no page
        // mapping).  Only if that fails, release the pool's unused memory to
        // the driver -- everything mapped again afterwards costs ~6 ms per GB
        // (measured: a config-5 contraction step 0.1 s -> 1.6 s after a full
        // trim).
        cudaGetLastError();
        trim_cache(0, s);
        cudaDeviceSynchronize();  // (the frees ran on the legacy stream)
        e = cudaMallocAsync(&p, bytes, s);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            int dev = 0;
            cudaMemPool_t pool;
            if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
                cudaMemPoolTrimTo(pool, 0);
            e = cudaMallocAsync(&p, bytes, s);
        }
    }
    LCC_CUDA(e);
    if (alloc_fill() >= 0) LCC_CUDA(cudaMemsetAsync(p, alloc_fill(), bytes, s));
    return p;
}

void* cache_alloc(size_t bytes, cudaStream_t s, size_t* cap) {
    Cache& c = cache();
    {
        std::lock_guard<std::mutex> g(c.m);
        auto it = c.free.lower_bound(bytes);
        if (it != c.free.end() && it->first <= 2 * bytes) {
            Block b = it->second;
            c.free.erase(it);
            c.held -= b.cap;
            if (b.s != s) cudaStreamWaitEvent(s, b.ready, 0);
            cudaEventDestroy(b.ready);
            *cap = b.cap;
            if (alloc_fill() >= 0) LCC_CUDA(cudaMemsetAsync(b.p, alloc_fill(), bytes, s));
            return b.p;
        }
    }
    const size_t want = (bytes + GRAIN - 1) / GRAIN * GRAIN;
    *cap = want;
    return pool_alloc(want, s);
}

void cache_free(void* p, size_t cap, cudaStream_t s) {
    Block b{p, cap, s, nullptr};
    if (cudaEventCreateWithFlags(&b.ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(b.ready, s) != cudaSuccess) {
        if (b.ready) cudaEventDestroy(b.ready);
        cudaFreeAsync(p, s);
        return;
    }
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.m);
    c.free.emplace(cap, b);
    c.held += cap;
}

void trim_cache(size_t keep_bytes, cudaStream_t) {
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.m);
    // drop the largest blocks first
    while (c.held > keep_bytes && !c.free.empty()) {
        auto it = std::prev(c.free.end());
        Block b = it->second;
        c.free.erase(it);
        c.held -= b.cap;
        // the releasing stream may be gone by now: wait for the block's last
        // use, then free on the legacy stream
        cudaEventSynchronize(b.ready);
        cudaEventDestroy(b.ready);
        cudaFreeAsync(b.p, 0);
    }
}

size_t cache_bytes() {
    Cache& c = cache();
    std::lock_guard<std::mutex> g(c.m);
    return c.held;
}

}  // namespace lcc
