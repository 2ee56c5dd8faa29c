// memory.cu -- device scratch allocation (see common.cuh: Buf).
//
// Large blocks (>= 1 MB) come from one arena per device, built on the CUDA
// virtual-memory API: a virtual range the size of the device is reserved
// once, physical memory is mapped at its end in >= 1 GB steps as the arena
// grows, and blocks are carved out of it best-fit with split and coalesce.
// Why not the stream-ordered pool (cudaMallocAsync) for these: mapping
// physical pages costs ~6 ms per GB on B200 -- more than the contraction
// that needs the buffer -- and the pool re-maps whenever a request does not
// fit a free virtual range; a cache of whole freed blocks on top of it
// (rounds 1-2) still fragmented at config 5 (3.6 G entries, ~150 GB of
// scratch per clustering): requests of a new size missed every cached block,
// ran the device out of memory, and the trim-and-retry path unmapped and
// re-mapped ~100 GB inside one clustering (2.7 s -> 5.9 s per call, run to
// run).  The arena never unmaps inside a call; every block of a call is
// scratch, so between calls the arena is one free range and is cut back
// from its end to the keep limit (LCC_POOL_KEEP_GB).
//
// Stream order: a block freed on stream t may be handed to stream s != t
// only after t's work up to the free; each stream's latest free is an
// event, and an allocation waits on the events of the other streams it has
// not yet seen (one stream in practice: no waits).
//
// The driver entry points (cuMem*) are fetched with cudaGetDriverEntryPoint,
// so the library has no link-time dependency on libcuda and still loads on
// a machine without a GPU.
#include <cuda.h>

#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace lcc {
namespace {

struct Driver {
    CUresult (*AddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
    CUresult (*Create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
    CUresult (*Map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
    CUresult (*SetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
    CUresult (*Unmap)(CUdeviceptr, size_t) = nullptr;
    CUresult (*Release)(CUmemGenericAllocationHandle) = nullptr;
    CUresult (*Granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
    bool ok = false;
};

const Driver& driver() {
    static Driver d = [] {
        Driver r;
        auto get = [](const char* name, void** fn) {
            cudaDriverEntryPointQueryResult q;
            return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
                   q == cudaDriverEntryPointSuccess && *fn != nullptr;
        };
        r.ok = get("cuMemAddressReserve", (void**)&r.AddressReserve) && get("cuMemCreate", (void**)&r.Create) &&
               get("cuMemMap", (void**)&r.Map) && get("cuMemSetAccess", (void**)&r.SetAccess) &&
               get("cuMemUnmap", (void**)&r.Unmap) && get("cuMemRelease", (void**)&r.Release) &&
               get("cuMemGetAllocationGranularity", (void**)&r.Granularity);
        if (getenv("LCC_ARENA") && getenv("LCC_ARENA")[0] == '0') r.ok = false;  // plain pool (diagnostics)
        cudaGetLastError();
        return r;
    }();
    return d;
}

constexpr size_t ALIGN = 1ull << 20;      // block sizes and offsets
constexpr size_t GROW_MIN = 1ull << 30;   // physical memory is mapped in steps of at least this

struct Arena {
    std::mutex m;
    int dev = -1;
    bool tried = false, ok = false;
    CUdeviceptr base = 0;
    size_t va = 0, mapped = 0, gran = 2ull << 20;
    struct Chunk { CUmemGenericAllocationHandle h; size_t off, size; };
    std::vector<Chunk> chunks;
    std::map<size_t, size_t> by_off;        // free blocks: offset -> size
    std::multimap<size_t, size_t> by_size;  //              size -> offset
    size_t free_bytes = 0;
    // stream order of reuse
    struct Freed { cudaEvent_t ev = nullptr; unsigned long long seq = 0; };
    std::map<cudaStream_t, Freed> freed;
    std::map<cudaStream_t, std::map<cudaStream_t, unsigned long long>> seen;

    void init() {
        tried = true;
        const Driver& d = driver();
        if (!d.ok) return;
        cudaFree(nullptr);  // a context on this device
        CUmemAllocationProp prop{};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = dev;
        if (d.Granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || gran == 0) return;
        size_t fr = 0, tot = 0;
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return;
        va = (tot + tot / 4 + gran - 1) / gran * gran;
        if (d.AddressReserve(&base, va, gran, 0, 0) != CUDA_SUCCESS) return;
        ok = true;
    }
    void erase_free(std::map<size_t, size_t>::iterator it) {
        auto r = by_size.equal_range(it->second);
        for (auto j = r.first; j != r.second; ++j)
            if (j->second == it->first) { by_size.erase(j); break; }
        free_bytes -= it->second;
        by_off.erase(it);
    }
    void insert_free(size_t off, size_t size) {
        // coalesce with the neighbours
        auto nx = by_off.lower_bound(off);
        if (nx != by_off.end() && off + size == nx->first) {
            size += nx->second;
            erase_free(nx);
        }
        nx = by_off.lower_bound(off);
        if (nx != by_off.begin()) {
            auto pv = std::prev(nx);
            if (pv->first + pv->second == off) {
                off = pv->first;
                size += pv->second;
                erase_free(pv);
            }
        }
        by_off.emplace(off, size);
        by_size.emplace(size, off);
        free_bytes += size;
    }
    // map at least `need` more bytes at the end of the arena
    bool grow(size_t need) {
        const Driver& d = driver();
        CUmemAllocationProp prop{};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = dev;
        CUmemAccessDesc acc{};
        acc.location = prop.location;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        const size_t exact = (need + gran - 1) / gran * gran;
        for (size_t sz : {std::max(exact, (GROW_MIN + gran - 1) / gran * gran), exact}) {
            if (mapped + sz > va) continue;
            CUmemGenericAllocationHandle h;
            if (d.Create(&h, sz, &prop, 0) != CUDA_SUCCESS) continue;
            if (d.Map(base + mapped, sz, 0, h, 0) != CUDA_SUCCESS) { d.Release(h); continue; }
            if (d.SetAccess(base + mapped, sz, &acc, 1) != CUDA_SUCCESS) {
                d.Unmap(base + mapped, sz);
                d.Release(h);
                continue;
            }
            chunks.push_back({h, mapped, sz});
            insert_free(mapped, sz);
            mapped += sz;
            return true;
        }
        return false;
    }
    void* take(size_t size, cudaStream_t s) {
        auto it = by_size.lower_bound(size);
        if (it == by_size.end()) return nullptr;
        const size_t bsz = it->first, off = it->second;
        erase_free(by_off.find(off));
        if (bsz > size) insert_free(off + size, bsz - size);
        // blocks freed on other streams: order this stream after those frees
        auto& sn = seen[s];
        for (auto& kv : freed) {
            if (kv.first == s) continue;
            unsigned long long& last = sn[kv.first];
            if (last < kv.second.seq) {
                cudaStreamWaitEvent(s, kv.second.ev, 0);
                last = kv.second.seq;
            }
        }
        return reinterpret_cast<void*>(base + off);
    }
    size_t trailing_free() const {
        if (by_off.empty()) return 0;
        auto last = std::prev(by_off.end());
        return last->first + last->second == mapped ? last->second : 0;
    }
    // unmap whole chunks from the end while more than `keep` bytes are mapped
    void trim(size_t keep) {
        bool synced = false;
        while (mapped > keep && !chunks.empty()) {
            const Chunk c = chunks.back();
            if (trailing_free() < c.size) break;
            if (!synced) {  // every free so far has completed before its memory goes away
                for (auto& kv : freed) cudaEventSynchronize(kv.second.ev);
                synced = true;
            }
            auto last = std::prev(by_off.end());
            const size_t off = last->first, size = last->second;
            erase_free(last);
            if (size > c.size) insert_free(off, size - c.size);
            driver().Unmap(base + c.off, c.size);
            driver().Release(c.h);
            chunks.pop_back();
            mapped -= c.size;
        }
    }
};

Arena& arena() {
    static Arena a[16];
    int dev = 0;
    cudaGetDevice(&dev);
    Arena& r = a[dev & 15];
    r.dev = dev;
    return r;
}

// diagnostics: LCC_ALLOC_FILL=<byte> fills every fresh scratch block, so a
// kernel that reads memory it never wrote shows up in every run
int alloc_fill() {
    static const int f = getenv("LCC_ALLOC_FILL") ? (int)strtol(getenv("LCC_ALLOC_FILL"), nullptr, 0) : -1;
    return f;
}

void trim_async_pool(size_t keep) {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
        cudaMemPoolTrimTo(pool, keep);
}

}  // namespace

// small buffers: the stream-ordered pool; one trim-and-retry
void* pool_alloc(size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        trim_cache(0, s);
        trim_async_pool(0);
        e = cudaMallocAsync(&p, bytes, s);
    }
    LCC_CUDA(e);
    if (alloc_fill() >= 0) LCC_CUDA(cudaMemsetAsync(p, alloc_fill(), bytes, s));
    return p;
}

void* cache_alloc(size_t bytes, cudaStream_t s, size_t* cap) {
    const size_t size = (bytes + ALIGN - 1) / ALIGN * ALIGN;
    *cap = size;
    Arena& a = arena();
    std::unique_lock<std::mutex> g(a.m);
    if (!a.tried) a.init();
    if (!a.ok) {
        g.unlock();
        return pool_alloc(size, s);
    }
    void* p = a.take(size, s);
    if (!p) {
        const size_t need = size - std::min(size, a.trailing_free());
        if (!a.grow(need)) {
            // hand the stream-ordered pool's unused memory back to the driver, then retry
            cudaDeviceSynchronize();
            trim_async_pool(0);
            if (!a.grow(need))
                throw OutOfMemory("device scratch: " + std::to_string(size >> 20) + " MB requested, " +
                                  std::to_string(a.mapped >> 20) + " MB mapped (" +
                                  std::to_string(a.free_bytes >> 20) + " MB of it free)");
        }
        p = a.take(size, s);
        if (!p) throw OutOfMemory("device scratch: arena fragmentation");
    }
    if (alloc_fill() >= 0) LCC_CUDA(cudaMemsetAsync(p, alloc_fill(), bytes, s));
    return p;
}

void cache_free(void* p, size_t cap, cudaStream_t s) {
    Arena& a = arena();
    std::lock_guard<std::mutex> g(a.m);
    if (!a.ok) {
        cudaFreeAsync(p, s);
        return;
    }
    Arena::Freed& f = a.freed[s];
    if (!f.ev) cudaEventCreateWithFlags(&f.ev, cudaEventDisableTiming);
    cudaEventRecord(f.ev, s);
    f.seq += 1;
    a.insert_free((size_t)(reinterpret_cast<CUdeviceptr>(p) - a.base), cap);
}

void trim_cache(size_t keep_bytes, cudaStream_t) {
    Arena& a = arena();
    std::lock_guard<std::mutex> g(a.m);
    if (a.ok) a.trim(keep_bytes);
}

size_t cache_bytes() {
    Arena& a = arena();
    std::lock_guard<std::mutex> g(a.m);
    return a.free_bytes;
}

void arena_bytes(size_t& mapped, size_t& free_bytes) {
    Arena& a = arena();
    std::lock_guard<std::mutex> g(a.m);
    mapped = a.mapped;
    free_bytes = a.free_bytes;
}

}  // namespace lcc
