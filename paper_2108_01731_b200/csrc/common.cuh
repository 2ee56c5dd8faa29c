// common.cuh -- shared helpers for the LambdaCC sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdexcept>
#include <string>

#include "../../include/lcc_b200.h"

namespace lcc {

// ---------------------------------------------------------------------------
// errors: thrown inside the library, converted to lcc_status at the C ABI.
// ---------------------------------------------------------------------------
struct Invalid : std::runtime_error { using std::runtime_error::runtime_error; };
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };
struct OutOfMemory : std::runtime_error { using std::runtime_error::runtime_error; };

#define LCC_CUDA(expr)                                                                  \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess) {                                                        \
            if (_e == cudaErrorMemoryAllocation)                                         \
                throw ::lcc::OutOfMemory(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
            throw ::lcc::CudaError(std::string(__FILE__) + ":" + std::to_string(__LINE__) + \
                                   " " #expr ": " + cudaGetErrorString(_e));            \
        }                                                                               \
    } while (0)

// Every launch of one of this library's kernels is followed by
// LCC_LAUNCH_CHECK(), which also counts it (lcc_kernel_launches()).
long long& launch_counter();
#define LCC_LAUNCH_CHECK()                     \
    do {                                       \
        ++::lcc::launch_counter();             \
        LCC_CUDA(cudaGetLastError());          \
    } while (0)

#define LCC_REQUIRE(cond, msg)                                                          \
    do { if (!(cond)) throw ::lcc::Invalid(msg); } while (0)

// ---------------------------------------------------------------------------
// device scratch.  Small buffers come straight from the stream-ordered pool
// (cudaMallocAsync).  Large ones (>= 1 MB: contraction keys/values, hub
// tables, per-round arrays at scale, the coarse levels) are carved out of a
// per-device arena of mapped virtual memory (memory.cu): mapping physical
// pages costs ~6 ms per GB on B200, so the arena keeps what it has mapped
// for the whole call and is cut back to the keep limit by trim_cache() when
// a C-ABI call returns.
// ---------------------------------------------------------------------------
constexpr size_t CACHE_MIN_BYTES = 1ull << 20;
void* cache_alloc(size_t bytes, cudaStream_t s, size_t* cap);
void cache_free(void* p, size_t cap, cudaStream_t s);
void trim_cache(size_t keep_bytes, cudaStream_t s);
size_t cache_bytes();

void* pool_alloc(size_t bytes, cudaStream_t s);  // cudaMallocAsync with one trim-and-retry

template <class T>
struct Buf {
    T* p = nullptr;
    size_t n = 0;
    size_t cap = 0;  // bytes actually held (cached blocks may be larger)
    cudaStream_t s = nullptr;
    Buf() = default;
    Buf(size_t count, cudaStream_t st) { alloc(count, st); }
    void alloc(size_t count, cudaStream_t st) {
        release();
        s = st;
        n = count;
        if (!count) return;
        const size_t bytes = sizeof(T) * count;
        if (bytes >= CACHE_MIN_BYTES) {
            p = static_cast<T*>(cache_alloc(bytes, st, &cap));
        } else {
            p = static_cast<T*>(pool_alloc(bytes, st));
            cap = bytes;
        }
    }
    void release() {
        if (p) {
            if (cap >= CACHE_MIN_BYTES) cache_free(p, cap, s);
            else cudaFreeAsync(p, s);
        }
        p = nullptr;
        n = 0;
        cap = 0;
    }
    ~Buf() { release(); }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    Buf(Buf&& o) noexcept : p(o.p), n(o.n), cap(o.cap), s(o.s) { o.p = nullptr; o.n = 0; o.cap = 0; }
    Buf& operator=(Buf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; cap = o.cap; s = o.s; o.p = nullptr; o.n = 0; o.cap = 0; }
        return *this;
    }
    T* get() const { return p; }
    operator T*() const { return p; }
};

// library scratch occupancy (GB mapped, GB in use): the arena of large
// blocks plus the stream-ordered pool of small ones; for traces and for the
// driver's does-the-contraction-fit estimate
void arena_bytes(size_t& mapped, size_t& free_bytes);
inline void pool_gb(double& reserved, double& used) {
    size_t am = 0, af = 0;
    arena_bytes(am, af);
    reserved = am / 1073741824.0;
    used = (am - af) / 1073741824.0;
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return;
    uint64_t r = 0, u = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &r);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &u);
    reserved += r / 1073741824.0;
    used += u / 1073741824.0;
}

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

inline unsigned grid_for(int64_t items, int block, int per_sm_cap = 8) {
    int64_t g = (items + block - 1) / block;
    int64_t cap = (int64_t)num_sms() * per_sm_cap;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
// Exact IEEE fp64 ops: the gain must be bit-identical to the oracle
// (gcc -ffp-contract=off), so no FMA contraction anywhere in the formula.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

// Exact u32 -> fp64 without I2F (the conversion runs on the narrow XU pipe,
// which ncu showed 56-70% busy in the table kernels): OR the integer into the
// mantissa of 2^52 and subtract 2^52 (exact for any 32-bit value).
__device__ __forceinline__ double u32_to_f64(uint32_t x) {
    return __dsub_rn(__hiloint2double(0x43300000, (int)x), 4503599627370496.0);
}

// Weight loads: WNone means every edge weighs 1.
// fsum: neighbour-cluster sums need floating point (float/double weights);
// otherwise they are exact integer sums in native 32-bit atomics (TW =
// uint32_t: 1 per edge unweighted, the count for LCC_W_U32).
struct WNone { };
template <class W> struct WLoad;
template <> struct WLoad<WNone> {
    static constexpr bool weighted = false, fsum = false;
    using TW = uint32_t;
    __device__ __forceinline__ static double at(const void*, int64_t) { return 1.0; }
    __device__ __forceinline__ static TW tw(const void*, int64_t) { return 1u; }
    __device__ __forceinline__ static double f64(TW x) { return u32_to_f64(x); }
};
template <> struct WLoad<uint32_t> {
    static constexpr bool weighted = true, fsum = false;
    using TW = uint32_t;
    __device__ __forceinline__ static TW tw(const void* w, int64_t e) {
        return __ldg(static_cast<const uint32_t*>(w) + e);
    }
    __device__ __forceinline__ static double at(const void* w, int64_t e) { return u32_to_f64(tw(w, e)); }
    __device__ __forceinline__ static double f64(TW x) { return u32_to_f64(x); }
};
template <> struct WLoad<float> {
    static constexpr bool weighted = true, fsum = true;
    using TW = double;
    __device__ __forceinline__ static double at(const void* w, int64_t e) {
        return (double)__ldg(static_cast<const float*>(w) + e);
    }
    __device__ __forceinline__ static TW tw(const void* w, int64_t e) { return at(w, e); }
    __device__ __forceinline__ static double f64(TW x) { return x; }
};
template <> struct WLoad<double> {
    static constexpr bool weighted = true, fsum = true;
    using TW = double;
    __device__ __forceinline__ static double at(const void* w, int64_t e) {
        return __ldg(static_cast<const double*>(w) + e);
    }
    __device__ __forceinline__ static TW tw(const void* w, int64_t e) { return at(w, e); }
    __device__ __forceinline__ static double f64(TW x) { return x; }
};

__device__ __forceinline__ double kval(const double* k, int64_t v) {
    return k ? __ldg(k + v) : 1.0;
}

// "a beats b": higher gain, ties to the lower cluster id.
__device__ __forceinline__ bool better(double ga, int32_t xa, double gb, int32_t xb) {
    return ga > gb || (ga == gb && (uint32_t)xa < (uint32_t)xb);
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// L2 eviction-priority policies (createpolicy, sm_80+): streamed CSR data is
// evict-first so it does not push the randomly gathered label / mass arrays
// out of the 126 MB L2; the gathered arrays are evict-last.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, %1;" : "=l"(p) : "f"(1.0f));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(p) : "f"(1.0f));
    return p;
}
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p, uint64_t pol) {
    int32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
// Random gathers ask L2 for 64 bytes per miss (LCC_PF64): a plain load's miss
// pulls a 128-byte line from DRAM on B200 -- measured 122.6 bytes of DRAM
// traffic per random 8-byte gather, 62.6 with .L2::64B (tools/micro/
// fetch_gran.cu, profiles/r02_fetch_gran.md) -- and nothing else of that
// line is wanted.
#ifndef LCC_GATHER64
#define LCC_GATHER64 1
#endif
#if LCC_GATHER64
#define LCC_PF64 ".L2::64B"
#else
#define LCC_PF64 ""
#endif
__device__ __forceinline__ int32_t ld_keep_i32(const int32_t* p, uint64_t pol) {
    int32_t r;
    asm volatile("ld.global.nc.L2::cache_hint" LCC_PF64 ".b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_keep_f64(const double* p, uint64_t pol) {
    double r;
    asm volatile("ld.global.nc.L2::cache_hint" LCC_PF64 ".f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
// read-only random gather without a cache policy (contraction, frontier)
__device__ __forceinline__ int32_t ld_gather_i32(const int32_t* p) {
    int32_t r;
    asm volatile("ld.global.nc" LCC_PF64 ".b32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31; }

constexpr int32_t EMPTY_KEY = -1;
constexpr int32_t NO_CAND = 0x7fffffff;

}  // namespace lcc
