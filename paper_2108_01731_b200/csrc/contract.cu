// contract.cu -- par_compress / par_flatten.
//
// Coarse ids: clusters are renumbered densely by ascending smallest-member
// id.  Labels are canonical (label == smallest member), so the root of every
// cluster is the vertex with C[x] == x and the coarse id is an exclusive scan
// of that flag.  Every directed CSR entry (v,u) is keyed (C'(v) << b | C'(u));
// intra-cluster entries get an all-ones sentinel (sorted last) and are summed
// into internal_offset.  A stable LSD radix sort over the 2b live key bits
// followed by a run-length reduce gives the coarse rows already sorted by
// neighbour id -- the same sort + segmented-sum contract as the reference's
// build_graph_arrays (graph.py:126-164).
#include <cub/cub.cuh>
#include <cstdio>
#include <type_traits>
#include <cstdlib>

#include "edgemap.cuh"
#include "internal.cuh"
#include "prims.cuh"

namespace lcc {
namespace {

struct IsRoot {
    const int32_t* C;
    int64_t n;
    __device__ __forceinline__ int32_t operator()(int32_t x) const { return (x < n && C[x] == x) ? 1 : 0; }
};

__global__ void k_map(const int32_t* __restrict__ C, const int32_t* __restrict__ rank,
                      const double* __restrict__ K, int64_t n, int32_t* mapping, double* ck) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = C[v];
        mapping[v] = rank[c];
        if (c == (int32_t)v) ck[rank[v]] = K[v];
    }
}

// Renumbering without the gather: rank(u) = #roots below u = the sampled scan
// at u's 32-vertex word + the popcount of the word's root bits below u.  For
// a root u, mapping[u] = rank(u); the two arrays are n/8 bytes together (L2
// resident at any size here) where mapping is 4n bytes of random gathers.
__global__ void k_rootbits(const int32_t* __restrict__ C, const int32_t* __restrict__ rank, int64_t n,
                           uint2* __restrict__ rb) {
    const int64_t nv = (n + 31) / 32 * 32;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nv; v += (int64_t)gridDim.x * blockDim.x) {
        const bool root = v < n && C[v] == (int32_t)v;
        const unsigned b = __ballot_sync(0xffffffffu, root);
        if ((v & 31) == 0) {
            rb[v >> 5] = make_uint2(b, (uint32_t)rank[v]);  // (bitmap word, roots before it): one 8-byte load per lookup
        }
    }
}
__device__ __forceinline__ int32_t root_rank(const uint2* __restrict__ rb, int32_t u) {
    const uint2 w = __ldg(rb + ((uint32_t)u >> 5));
    return (int32_t)(w.y + __popc(w.x & ((1u << (u & 31)) - 1u)));
}

// edge functor: key of the directed entry (v, u), intra entries -> sentinel
template <class WT, class VT>
struct EdgeKey {
    const int32_t* indices;
    const void* w;
    const int32_t* mapping;
    int bits;
    uint64_t sentinel;
    uint64_t* keys;
    VT* vals;
    unsigned long long* intra_cnt;
    double* intra_w;
    bool compact = false;  // write at the list position (complex rows only) instead of the CSR index
    unsigned long long cnt = 0;
    double acc = 0.0;
    // two-phase (edgemap.cuh): a thread's gathers all go out before its first store;
    // the per-thread sums keep their element order
    struct Tmp { uint32_t a, b; typename WLoad<WT>::TW wv; };
    __device__ __forceinline__ Tmp load(int64_t v, int64_t e, int64_t) const {
        return Tmp{(uint32_t)__ldg(mapping + v), (uint32_t)ld_gather_i32(mapping + __ldg(indices + e)), WLoad<WT>::tw(w, e)};
    }
    __device__ __forceinline__ void store(const Tmp& t, int64_t, int64_t e, int64_t pos) {
        const uint64_t a = t.a, b = t.b;
        const auto wv = t.wv;
        const int64_t o = compact ? pos : e;
        if (a == b) {
            keys[o] = sentinel;
            ++cnt;
            acc += WLoad<WT>::f64(wv);
        } else {
            keys[o] = (a << bits) | b;
        }
        if (vals) vals[o] = (VT)wv;
    }
    __device__ __forceinline__ void flush() {
        for (int d = 16; d; d >>= 1) {
            cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
            acc += __shfl_xor_sync(0xffffffffu, acc, d);
        }
        if ((threadIdx.x & 31) == 0 && cnt) {
            atomicAdd(intra_cnt, cnt);
            atomicAdd(intra_w, acc);
        }
    }
};

__global__ void k_emit_rows(const uint64_t* __restrict__ ukeys, int64_t R, int bits, int64_t cn,
                            int64_t* cindptr, int32_t* cindices) {
    const uint64_t mask = (1ULL << bits) - 1ULL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= R; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i < R ? (int64_t)(ukeys[i] >> bits) : cn;
        const int64_t prev = i > 0 ? (int64_t)(ukeys[i - 1] >> bits) : -1;
        for (int64_t r = prev + 1; r <= row; ++r) cindptr[r] = i;
        if (i < R) cindices[i] = (int32_t)(ukeys[i] & mask);
    }
}

struct Sq {
    __device__ __forceinline__ double operator()(double x) const { return x * x; }
};
struct U32F64 {
    __device__ __forceinline__ double operator()(uint32_t x) const { return (double)x; }
};
struct KSq {
    const double* k;
    __device__ __forceinline__ double operator()(int64_t v) const { const double x = k ? k[v] : 1.0; return x * x; }
};

struct RunHead {
    const uint64_t* keys;
    __device__ __forceinline__ int64_t operator()(int64_t i) const {
        return (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
    }
};

// LCC_TRACE: device time of each contraction phase on stderr
struct PhaseTrace {
    cudaStream_t s;
    bool on;
    cudaEvent_t last = nullptr;
    explicit PhaseTrace(cudaStream_t st) : s(st), on(getenv("LCC_TRACE") != nullptr) {
        if (on) { cudaEventCreate(&last); cudaEventRecord(last, s); }
    }
    void mark(const char* what) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, s);
        cudaEventSynchronize(e);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, last, e);
        double r, u;
        pool_gb(r, u);
        fprintf(stderr, "[lcc]     compress %-10s %.2f ms  (pool %.1f GB reserved, %.1f used)\n", what, ms, r, u);
        cudaEventDestroy(last);
        last = e;
    }
    ~PhaseTrace() { if (last) cudaEventDestroy(last); }
};

// ---- fast path: most clusters are singletons ------------------------------
// A fine row u is "simple" when u is a singleton cluster and none of its
// neighbours lies in a non-singleton cluster: its coarse row is the fine row
// with every id mapped (strictly increasing -- the renumbering is monotone on
// singletons -- and duplicate free) and the same weights.  Only the other
// ("complex") rows go through keys + radix sort + reduce; the simple ones are
// copied by one streaming pass.  Complex rows = members of non-singleton
// clusters and their neighbours (one edge pass over the members' rows).  The
// output is identical to the full path's (same rows, same per-entry sums in
// the same order).  Config 4: the level 1 -> 2 contraction merges 6 of 14.6M
// vertices, and its 506M-entry radix sort was 60% of that level's time.
__global__ void k_csize(const int32_t* __restrict__ mapping, int64_t n, int32_t* csize) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(csize + mapping[v], 1);
}
__global__ void k_members(const int32_t* __restrict__ mapping, const int32_t* __restrict__ csize, int64_t n,
                          uint8_t* cf) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        cf[v] = csize[mapping[v]] > 1 ? 1 : 0;
}
struct MarkNbrs {
    const int32_t* indices;
    uint8_t* cf;
    __device__ __forceinline__ void operator()(int64_t, int64_t e, int64_t) { cf[__ldg(indices + e)] = 1; }
    __device__ __forceinline__ void flush() {}
};
struct DegOf {
    const int64_t* indptr;
    const int32_t* list;
    int64_t n;
    __device__ __forceinline__ int64_t operator()(int64_t i) const {
        if (i >= n) return 0;
        const int32_t v = list[i];
        return indptr[v + 1] - indptr[v];
    }
};
__global__ void k_simple_len(const int64_t* __restrict__ indptr, const uint8_t* __restrict__ cf,
                             const int32_t* __restrict__ mapping, int64_t n, int64_t* clen) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if (!cf[v]) clen[mapping[v]] = indptr[v + 1] - indptr[v];
}
// run starts, then run ends (two passes: no thread walks a hub's long row)
__global__ void k_complex_start(const uint64_t* __restrict__ ukeys, int64_t R, int bits, int64_t* cstart) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = (int64_t)(ukeys[i] >> bits);
        if (i == 0 || (int64_t)(ukeys[i - 1] >> bits) != row) cstart[row] = i;
    }
}
__global__ void k_complex_len(const uint64_t* __restrict__ ukeys, int64_t R, int bits, const int64_t* cstart,
                              int64_t* clen) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = (int64_t)(ukeys[i] >> bits);
        if (i == R - 1 || (int64_t)(ukeys[i + 1] >> bits) != row) clen[row] = i + 1 - cstart[row];
    }
}
template <class WT, class OT>
struct EmitSimple {
    const int32_t* indices;
    const void* w;
    const int32_t* mapping;
    const uint8_t* cf;
    const int64_t* indptr;
    const int64_t* cindptr;
    int32_t* cind;
    OT* cw;
    const uint2* rb;        // every neighbour of a simple row is a root: its
                            // coarse id is its rank (no mapping gather).  Null
                            // for a shard's partial rows: a neighbour whose row
                            // lives on another rank never marked this row, so
                            // it may be a non-root; those rows keep the gather
                            // (the owner-side merge sorts and sums them)
    struct Tmp { int32_t id; OT wv; };  // (the output position is recomputed in store(): 72 -> fewer registers, 3 -> more CTAs per SM)
    // per row: where its entries go (output position = that + e), or "not a simple row"
    __device__ __forceinline__ int64_t prep(int64_t v) const {
        return cf[v] ? INT64_MIN : cindptr[mapping[v]] - __ldg(indptr + v);
    }
    __device__ __forceinline__ Tmp load(int64_t aux, int64_t e, int64_t) const {
        Tmp t;
        t.id = 0;
        t.wv = OT(0);
        if (aux == INT64_MIN) return t;
        const int32_t u = __ldg(indices + e);
        t.id = rb ? root_rank(rb, u) : ld_gather_i32(mapping + u);
        t.wv = (OT)WLoad<WT>::tw(w, e);
        return t;
    }
    __device__ __forceinline__ void store(const Tmp& t, int64_t aux, int64_t e, int64_t) const {
        if (aux == INT64_MIN) return;
        cind[aux + e] = t.id;
        cw[aux + e] = t.wv;
    }
    __device__ __forceinline__ void flush() {}
};
template <class OT, class ST>
__global__ void k_emit_complex(const uint64_t* __restrict__ ukeys, const ST* __restrict__ sums, int64_t R, int bits,
                               const int64_t* __restrict__ cindptr, const int64_t* __restrict__ cstart,
                               int32_t* cind, OT* cw) {
    const uint64_t mask = (1ULL << bits) - 1ULL;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = (int64_t)(ukeys[i] >> bits);
        const int64_t o = cindptr[row] + (i - cstart[row]);
        cind[o] = (int32_t)(ukeys[i] & mask);
        cw[o] = (OT)sums[i];
    }
}

// ---- segmented contraction (integer sums; LCC_CONTRACT_SEG, default on) --
// The fine entries are laid out coarse row by coarse row -- vertices sorted
// by (coarse id, id) with one radix sort of n 32-bit keys, then an
// edge-balanced pass writes each entry's coarse neighbour (or an intra
// sentinel) at its row's position -- so only each coarse row has to be
// sorted, not the whole 64-bit key space:
//   * rows of <= SEG_MAX entries: windows of consecutive rows (<= 4096
//     entries) sorted in one CTA (cub::BlockRadixSort on (row offset, id),
//     12 + b bits), duplicates summed in shared memory, written back in place;
//   * longer rows (hubs): one device radix sort of (row, id) keys over their
//     entries only, reduce-by-key, scattered back in place;
//   * a scan of the per-row unique counts and one copy give the exact-size
//     coarse CSR.  Integer sums are exact in any order: the output equals the
//     global-sort path entry for entry.
#ifndef LCC_SEG_T
#define LCC_SEG_T 256
#endif
#ifndef LCC_SEG_I
#define LCC_SEG_I 16
#endif
#ifndef LCC_SEG_MINB
#define LCC_SEG_MINB 2  // 2 CTAs per SM (128 registers): with 1 the compiler took more registers and the windows ran 30% slower
#endif
constexpr int SEG_T = LCC_SEG_T, SEG_I = LCC_SEG_I, SEG_CAP = SEG_T * SEG_I;  // entries per window CTA
#ifndef LCC_SEG_WIN
#define LCC_SEG_WIN 3072
#endif
#ifndef LCC_SEG_MAXROW
#define LCC_SEG_MAXROW 1024
#endif
// window = rows starting in [w*WIN, (w+1)*WIN); rows over SEG_MAX entries are sorted on their own (k_seg_row, device
// sort).  A window holds up to WIN + MAX <= SEG_CAP entries and the CTA sorts SEG_CAP keys whatever it holds: 3072 +
// 1024 fills ~80% of them, 2048 + 2048 filled ~55% (config 5 level 0: windows 121 -> see DESIGN ms)
constexpr int64_t SEG_WIN = LCC_SEG_WIN;
constexpr int64_t SEG_MAX = LCC_SEG_MAXROW;
static_assert(SEG_WIN + SEG_MAX <= SEG_CAP, "a window must fit one CTA sort");
constexpr uint32_t SEG_SENT = 0xffffffffu;
#ifndef LCC_SEG_RADIX_BITS
#define LCC_SEG_RADIX_BITS 5  // window sorts: 8 passes over 12 + b bits instead of 10 (config 5 level 0: 196 -> 176 ms)
#endif

__global__ void k_seg_keys(const int32_t* __restrict__ mapping, int64_t n, uint32_t* keys, int32_t* ids) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        keys[v] = (uint32_t)mapping[v];
        ids[v] = (int32_t)v;
    }
}
struct DegPerm {
    const int64_t* indptr;
    const int32_t* perm;
    int64_t n;
    __device__ __forceinline__ int64_t operator()(int64_t i) const {
        if (i >= n) return 0;
        const int32_t v = perm[i];
        return indptr[v + 1] - indptr[v];
    }
};
__global__ void k_seg_rstart(const uint32_t* __restrict__ skeys, const int64_t* __restrict__ pos0, int64_t n,
                             int64_t cn, int64_t* rstart) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (i == 0 || skeys[i] != skeys[i - 1]) rstart[skeys[i]] = pos0[i];
        if (i == 0) rstart[cn] = pos0[n];
    }
}
template <class WT>
struct SegFill {
    const int32_t* indices;
    const void* w;
    const int32_t* mapping;
    uint32_t* keys;
    uint32_t* vals;
    unsigned long long* intra;
    // optional (LCC_SEG_FILLBITS=1, measured slower): a root's coarse id is
    // its rank among the roots, read from the root bitmap and its sampled
    // prefix (2 x n/8 bytes, L2 resident) instead of the n-word mapping
    const uint2* rb;
    unsigned long long cnt = 0;
#ifndef LCC_FILL_TWOPHASE
#define LCC_FILL_TWOPHASE 1
#endif
#if LCC_FILL_TWOPHASE
    struct Tmp { int32_t a, b; uint32_t wv; };
#else
    struct Tmp1 { int32_t a, b; uint32_t wv; };
    using Tmp_ = Tmp1;
    __device__ __forceinline__ void operator()(int64_t v, int64_t e, int64_t pos) { store(load(v, e, pos), v, e, pos); }
#endif
#if LCC_FILL_TWOPHASE
    using Tmp_ = Tmp;
#endif
    __device__ __forceinline__ Tmp_ load(int64_t v, int64_t e, int64_t) const {
        Tmp_ t;
        t.a = __ldg(mapping + v);
        const int32_t u = __ldg(indices + e);
        if (rb) {
            const uint2 wd = __ldg(rb + ((uint32_t)u >> 5));
            if ((wd.x >> (u & 31)) & 1u) t.b = (int32_t)(wd.y + __popc(wd.x & ((1u << (u & 31)) - 1u)));
            else t.b = ld_gather_i32(mapping + u);
        } else {
            t.b = ld_gather_i32(mapping + u);
        }
        t.wv = WLoad<WT>::tw(w, e);
        return t;
    }
    __device__ __forceinline__ void store(const Tmp_& t, int64_t, int64_t, int64_t pos) {
        if (t.a == t.b) {
            keys[pos] = SEG_SENT;
            cnt += t.wv;
        } else {
            keys[pos] = (uint32_t)t.b;
        }
        vals[pos] = t.wv;
    }
    __device__ __forceinline__ void flush() {
        for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
        if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(intra, cnt);
    }
};
// first row of each window: lower bound of w*WIN in rstart
__global__ void k_seg_wrow(const int64_t* __restrict__ rstart, int64_t cn, int64_t nwin, int64_t* wrow) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w <= nwin; w += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = w * SEG_WIN;
        int64_t lo = 0, hi = cn;  // first a in [0, cn) with rstart[a] >= t, else cn
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (rstart[mid] < t) lo = mid + 1; else hi = mid;
        }
        wrow[w] = lo;
    }
}
struct MaxOp {
    __device__ __forceinline__ int operator()(int a, int b) const { return a > b ? a : b; }
};
struct SegSmem {
    using Sort64 = cub::BlockRadixSort<uint64_t, SEG_T, SEG_I, uint32_t, LCC_SEG_RADIX_BITS>;
    using Sort32 = cub::BlockRadixSort<uint32_t, SEG_T, SEG_I, uint32_t, LCC_SEG_RADIX_BITS>;
    using ScanI = cub::BlockScan<int, SEG_T>;
    using ScanU = cub::BlockScan<uint32_t, SEG_T>;
    union {
        typename Sort64::TempStorage sort64;
        typename Sort32::TempStorage sort32;
        typename ScanI::TempStorage scani;
        typename ScanU::TempStorage scanu;
        uint64_t key[SEG_CAP];
    } u;
    int32_t rid[SEG_CAP];     // row id at its start offset, -1 elsewhere
    uint32_t runbase[SEG_CAP];
    // per row of the window (at most SEG_WIN non-empty rows start in it)
    int32_t roff[SEG_WIN];    // start offset
    int32_t hexrow[SEG_WIN];  // exclusive head (run) count at its start
    int32_t cnt[SEG_WIN];     // unique entries
};
// One window: keys are (row number inside the window, coarse id).  A window
// of ~2048 entries holds a few dozen rows, so the pair usually fits 32 bits
// (b + 5-6 bits: 6 passes of 5-bit digits on 32-bit keys instead of 8 on
// 64-bit ones; config-5 level 0: 176 -> see DESIGN ms); windows of many short
// rows keep 64-bit keys.
template <class KeyT>
__device__ __forceinline__ void seg_window_body(SegSmem& sm, int64_t base, int T, int nrows, int bbits, int rbits,
                                                const int (&ridx)[SEG_I], uint32_t* keys, uint32_t* vals) {
    const uint32_t bmask = (uint32_t)((1ull << bbits) - 1ull);
    KeyT key[SEG_I];
    uint32_t val[SEG_I];
#pragma unroll
    for (int j = 0; j < SEG_I; ++j) {
        const int i = threadIdx.x * SEG_I + j;
        if (i < T) {
            // a row over SEG_MAX entries that starts inside the window is left to the row
            // kernels: its entries count as dead here (nothing of it is written)
            const int rn = ridx[j];
            const bool longrow = (rn + 1 < nrows ? sm.roff[rn + 1] : T) - sm.roff[rn] > (int)SEG_MAX;
            const uint32_t b = keys[base + i];
            key[j] = ((KeyT)rn << bbits) | (KeyT)((b == SEG_SENT || longrow) ? bmask : b);
            val[j] = vals[base + i];
        } else {
            key[j] = (KeyT)~(KeyT)0;
            val[j] = 0u;
        }
    }
    // (padding keys are all ones: beyond every live key on the sorted bits or tied with the
    // last row's sentinel; either way they end up at positions >= T or among the dead entries)
    if constexpr (sizeof(KeyT) == 8) SegSmem::Sort64(sm.u.sort64).Sort(key, val, 0, rbits + bbits);
    else SegSmem::Sort32(sm.u.sort32).Sort(key, val, 0, rbits + bbits);
    __syncthreads();
    KeyT* skey = reinterpret_cast<KeyT*>(sm.u.key);
#pragma unroll
    for (int j = 0; j < SEG_I; ++j) skey[threadIdx.x * SEG_I + j] = key[j];
    __syncthreads();
    int head[SEG_I], hx[SEG_I];
    bool endf[SEG_I];
#pragma unroll
    for (int j = 0; j < SEG_I; ++j) {
        const int i = threadIdx.x * SEG_I + j;
        const bool live = i < T && key[j] != (KeyT)~(KeyT)0 && (uint32_t)(key[j] & (KeyT)bmask) != bmask;
        head[j] = live && (i == 0 || skey[i - 1] != key[j]);
        endf[j] = live && (i == T - 1 || skey[i + 1] != key[j]);
    }
    __syncthreads();  // the key array is reused by the scans below
    SegSmem::ScanI(sm.u.scani).ExclusiveSum(head, hx);
    __syncthreads();
    uint32_t pw[SEG_I];
    SegSmem::ScanU(sm.u.scanu).InclusiveSum(val, pw);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SEG_I; ++j) {
        const int i = threadIdx.x * SEG_I + j;
        if (i < T && sm.rid[i] >= 0) sm.hexrow[ridx[j]] = hx[j];  // sorted rows keep their extents
        if (head[j]) {
            sm.runbase[hx[j]] = pw[j] - val[j];
            atomicAdd(&sm.cnt[(int)(key[j] >> bbits)], 1);
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SEG_I; ++j) {
        if (!endf[j]) continue;
        const int r = hx[j] + head[j] - 1;  // this run's number
        const int rown = (int)(key[j] >> bbits);
        const int64_t out = base + sm.roff[rown] + (r - sm.hexrow[rown]);
        keys[out] = (uint32_t)(key[j] & (KeyT)bmask);
        vals[out] = pw[j] - sm.runbase[r];
    }
}
__global__ void __launch_bounds__(SEG_T, LCC_SEG_MINB)
k_seg_window(const int64_t* __restrict__ rstart, const int64_t* __restrict__ wrow, int64_t nwin, int bbits, int key64,
             uint32_t* keys, uint32_t* vals, int32_t* ucnt) {
    extern __shared__ __align__(16) unsigned char smraw[];
    SegSmem& sm = *reinterpret_cast<SegSmem*>(smraw);
    for (int64_t w = blockIdx.x; w < nwin; w += gridDim.x) {
        const int64_t r0 = wrow[w], r1 = wrow[w + 1];
        if (r0 >= r1) continue;
        const int64_t rlast = r1 - 1;
        const int64_t rend = (rstart[rlast + 1] - rstart[rlast] > SEG_MAX) ? rlast : r1;
        const int64_t base = rstart[r0];
        const int T = (int)(rstart[rend] - base);
        if (T <= 0) continue;
        for (int i = threadIdx.x; i < SEG_CAP; i += SEG_T) sm.rid[i] = -1;
        for (int i = threadIdx.x; i < (int)SEG_WIN; i += SEG_T) sm.cnt[i] = 0;
        __syncthreads();
        for (int64_t a = r0 + threadIdx.x; a < rend; a += SEG_T)
            if (rstart[a + 1] > rstart[a]) sm.rid[rstart[a] - base] = (int32_t)a;
        __syncthreads();
        // row number of every position: inclusive count of the row starts - 1
        int ridx[SEG_I];
#pragma unroll
        for (int j = 0; j < SEG_I; ++j) {
            const int i = threadIdx.x * SEG_I + j;
            ridx[j] = (i < T && sm.rid[i] >= 0) ? 1 : 0;
        }
        int nrows = 0;
        SegSmem::ScanI(sm.u.scani).InclusiveSum(ridx, ridx, nrows);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < SEG_I; ++j) {
            const int i = threadIdx.x * SEG_I + j;
            ridx[j] -= 1;
            if (i < T && sm.rid[i] >= 0) sm.roff[ridx[j]] = i;
        }
        __syncthreads();
        const int rbits = 32 - __clz(max(nrows - 1, 1));
        if (!key64 && rbits + bbits <= 32) seg_window_body<uint32_t>(sm, base, T, nrows, bbits, rbits, ridx, keys, vals);
        else seg_window_body<uint64_t>(sm, base, T, nrows, bbits, rbits, ridx, keys, vals);
        __syncthreads();
        for (int k = threadIdx.x; k < nrows; k += SEG_T)
            if ((k + 1 < nrows ? sm.roff[k + 1] : T) - sm.roff[k] <= (int)SEG_MAX) ucnt[sm.rid[sm.roff[k]]] = sm.cnt[k];
        __syncthreads();
    }
}
// Rows of (SEG_MAX, THREADS * ITEMS] entries: one CTA sorts one row on the b
// bits of the coarse ids alone (5 passes of 5-bit digits at config 5 instead
// of the windows' 8 over (row offset, id), and no 64-bit device sort of
// (row, id) keys: config-5 level 0, rows of 2049-8192 entries hold ~9% of the
// entries and took 81 ms there).  Same run logic as k_seg_window with a
// single row: sentinels (and the padding) sort last, duplicate ids are summed
// from an inclusive scan of the sorted weights, the row's unique entries are
// written back in place from its start.
constexpr int64_t SEG_ROW_MAX = 8192;
template <int THREADS, int ITEMS>
struct RowSmem {
    static constexpr int CAP = THREADS * ITEMS;
    using Sort = cub::BlockRadixSort<uint32_t, THREADS, ITEMS, uint32_t, LCC_SEG_RADIX_BITS>;
    using ScanI = cub::BlockScan<int, THREADS>;
    using ScanU = cub::BlockScan<uint32_t, THREADS>;
    union {
        typename Sort::TempStorage sort;
        typename ScanI::TempStorage scani;
        typename ScanU::TempStorage scanu;
        uint32_t key[CAP];
    } u;
    uint32_t runbase[CAP];
};
template <int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS)
k_seg_row(const int64_t* __restrict__ rstart, const int32_t* __restrict__ rows, int64_t nrows, int bbits,
          uint32_t* keys, uint32_t* vals, int32_t* ucnt) {
    using SM = RowSmem<THREADS, ITEMS>;
    extern __shared__ __align__(16) unsigned char smraw[];
    SM& sm = *reinterpret_cast<SM*>(smraw);
    const uint32_t bmask = (uint32_t)((1ull << bbits) - 1ull);
    for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
        const int32_t a = rows[r];
        const int64_t base = rstart[a];
        const int T = (int)(rstart[a + 1] - base);
        uint32_t key[ITEMS], val[ITEMS];
        // striped loads (coalesced), then into the blocked arrangement the sort wants
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int i = j * THREADS + threadIdx.x;
            uint32_t b = bmask, w = 0u;
            if (i < T) {
                b = keys[base + i];
                if (b == SEG_SENT) b = bmask;
                w = vals[base + i];
            }
            key[j] = b;
            val[j] = w;
        }
        typename SM::Sort(sm.u.sort).Sort(key, val, 0, bbits);  // any arrangement in: a full sort follows
        __syncthreads();
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) sm.u.key[threadIdx.x * ITEMS + j] = key[j];
        __syncthreads();
        int head[ITEMS], hx[ITEMS];
        bool endf[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const int i = threadIdx.x * ITEMS + j;
            const bool live = key[j] != bmask;  // sentinels and padding sort last
            head[j] = live && (i == 0 || sm.u.key[i - 1] != key[j]);
            endf[j] = live && (i == SM::CAP - 1 || sm.u.key[i + 1] != key[j]);
        }
        __syncthreads();  // the key array is reused by the scans below
        int nruns = 0;
        typename SM::ScanI(sm.u.scani).ExclusiveSum(head, hx, nruns);
        __syncthreads();
        uint32_t pw[ITEMS];
        typename SM::ScanU(sm.u.scanu).InclusiveSum(val, pw);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < ITEMS; ++j)
            if (head[j]) sm.runbase[hx[j]] = pw[j] - val[j];
        __syncthreads();
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            if (!endf[j]) continue;
            const int run = hx[j] + head[j] - 1;
            keys[base + run] = key[j];
            vals[base + run] = pw[j] - sm.runbase[run];
        }
        if (threadIdx.x == 0) ucnt[a] = nruns;
        __syncthreads();
    }
}
struct RowLenIn {
    const int64_t* rstart;
    int64_t lo, hi;  // (lo, hi]
    __device__ __forceinline__ bool operator()(int32_t a) const {
        const int64_t L = rstart[a + 1] - rstart[a];
        return L > lo && L <= hi;
    }
};
template <int THREADS, int ITEMS>
void seg_rows(const int64_t* rstart, int64_t cn, int64_t lo, int bbits, uint32_t* keys, uint32_t* vals, int32_t* ucnt,
              cudaStream_t s) {
    using SM = RowSmem<THREADS, ITEMS>;
    Buf<int32_t> rows(std::max<int64_t>(cn, 1), s);
    Buf<int64_t> dn(1, s);
    select_if(cub::CountingInputIterator<int32_t>(0), rows.get(), dn.get(), cn, RowLenIn{rstart, lo, (int64_t)SM::CAP}, s);
    int64_t nr = 0;
    LCC_CUDA(cudaMemcpyAsync(&nr, dn.get(), sizeof(nr), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    if (nr == 0) return;
    if (getenv("LCC_TRACE")) fprintf(stderr, "[lcc]     compress seg rows of (%lld, %d] entries: %lld\n", (long long)lo, SM::CAP, (long long)nr);
    const int SMEM = (int)sizeof(SM);
    static int occ = 0;
    if (!occ) {
        LCC_CUDA(cudaFuncSetAttribute(k_seg_row<THREADS, ITEMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
        LCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_seg_row<THREADS, ITEMS>, THREADS, SMEM));
        occ = std::max(occ, 1);
    }
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nr, (int64_t)num_sms() * occ));
    k_seg_row<THREADS, ITEMS><<<grid, THREADS, SMEM, s>>>(rstart, rows.get(), nr, bbits, keys, vals, ucnt);
    LCC_LAUNCH_CHECK();
}
struct RowLenBig {
    const int64_t* rstart;
    int64_t lim;
    __device__ __forceinline__ bool operator()(int32_t a) const { return rstart[a + 1] - rstart[a] > lim; }
};
struct BigLen {
    const int64_t* rstart;
    const int32_t* list;
    int64_t nb;
    __device__ __forceinline__ int64_t operator()(int64_t i) const {
        if (i >= nb) return 0;
        const int32_t a = list[i];
        return rstart[a + 1] - rstart[a];
    }
};
// keys of the long rows: (rank of the row among the long rows, coarse id) --
// a few 10K rows, so ~40 live bits (5 radix passes) instead of 2b (7)
__global__ void k_big_rank(const int32_t* __restrict__ big, int64_t nb, int32_t* __restrict__ brank) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.x * blockDim.x)
        brank[big[i]] = (int32_t)i;
}
struct BigKeys {
    const uint32_t* keys;
    const uint32_t* vals;
    const int32_t* brank;
    int bbits;
    uint64_t* k64;
    uint32_t* v32;
    struct Tmp { uint32_t b, v; int32_t rk; };
    __device__ __forceinline__ Tmp load(int64_t a, int64_t e, int64_t) const { return Tmp{keys[e], vals[e], __ldg(brank + a)}; }
    __device__ __forceinline__ void store(const Tmp& t, int64_t, int64_t, int64_t pos) const {
        const uint32_t bmask = (uint32_t)((1ull << bbits) - 1ull);
        k64[pos] = ((uint64_t)t.rk << bbits) | (t.b == SEG_SENT ? bmask : t.b);
        v32[pos] = t.v;
    }
    __device__ __forceinline__ void flush() {}
};
__global__ void k_big_first(const uint64_t* __restrict__ uk, const int64_t* __restrict__ nruns, int bbits,
                            int64_t* first) {
    const int64_t R = *nruns;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = (int64_t)(uk[i] >> bbits);
        if (i == 0 || (int64_t)(uk[i - 1] >> bbits) != a) first[a] = i;
    }
}
__global__ void k_big_emit(const uint64_t* __restrict__ uk, const uint32_t* __restrict__ us,
                           const int64_t* __restrict__ nruns, int bbits, const int64_t* __restrict__ first,
                           const int32_t* __restrict__ big, const int64_t* __restrict__ rstart, uint32_t* keys,
                           uint32_t* vals, int32_t* ucnt) {
    const int64_t R = *nruns;
    const uint32_t bmask = (uint32_t)((1ull << bbits) - 1ull);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < R; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rk = (int64_t)(uk[i] >> bbits);
        const int64_t a = big[rk];
        const uint32_t b = (uint32_t)(uk[i] & bmask);
        if (b == bmask) continue;  // intra sentinel (sorts last in its row)
        const int64_t out = rstart[a] + (i - first[rk]);
        keys[out] = b;
        vals[out] = us[i];
        atomicAdd(ucnt + a, 1);
    }
}
struct SegCopy {
    const uint32_t* keys;
    const uint32_t* vals;
    int32_t* cind;
    uint32_t* cw;
    struct Tmp { uint32_t k, v; };
    __device__ __forceinline__ Tmp load(int64_t, int64_t e, int64_t) const { return Tmp{keys[e], vals[e]}; }
    __device__ __forceinline__ void store(const Tmp& t, int64_t, int64_t, int64_t pos) const {
        cind[pos] = (int32_t)t.k;
        cw[pos] = t.v;
    }
    __device__ __forceinline__ void flush() {}
};

// coarse CSR of an integer-weighted graph by the segmented path; fills
// out.indptr/indices/wi, returns the entry count; *intra = intra weight
template <class WT>
int64_t compress_seg(const lcc_graph& g, const int32_t* mapping, int64_t cn, Coarse& out, unsigned long long* intra,
                     const uint2* rb, cudaStream_t s) {
    const int64_t n = g.n, nnz = g.nnz;
    const int bbits = std::max(1, bit_width((uint64_t)cn));
    LCC_REQUIRE(bbits <= 31, "coarse graph too large for the segmented contraction");
    PhaseTrace tr(s);
    // 1. vertices in (coarse id, id) order, their rows' positions
    Buf<int64_t> pos0(n + 1, s), rstart(cn + 1, s);
    Buf<int32_t> perm(n, s);
    Buf<uint32_t> skeys(n, s);
    {
        Buf<uint32_t> k0(n, s);
        Buf<int32_t> ids(n, s);
        k_seg_keys<<<grid_for(n, 256), 256, 0, s>>>(mapping, n, k0.get(), ids.get());
        LCC_LAUNCH_CHECK();
        size_t bytes = 0;
        LCC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0.get(), skeys.get(), ids.get(), perm.get(), n, 0,
                                                 bbits, s));
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), bytes, k0.get(), skeys.get(), ids.get(), perm.get(), n,
                                                 0, bbits, s));
    }
    cub::TransformInputIterator<int64_t, DegPerm, cub::CountingInputIterator<int64_t>> degs(
        cub::CountingInputIterator<int64_t>(0), DegPerm{g.indptr, perm.get(), n});
    exclusive_sum(degs, pos0.get(), n + 1, s);
    k_seg_rstart<<<grid_for(n, 256), 256, 0, s>>>(skeys.get(), pos0.get(), n, cn, rstart.get());
    LCC_LAUNCH_CHECK();
    skeys.release();
    tr.mark("seg order");
    // 2. every entry's coarse neighbour at its row position
    Buf<uint32_t> keys(nnz, s), vals(nnz, s);
    edge_balanced(g.indptr, perm.get(), pos0.get(), n, nnz,
                  SegFill<WT>{g.indices, g.weights, mapping, keys.get(), vals.get(), intra, rb}, s);
    perm.release();
    pos0.release();
    tr.mark("seg fill");
    // 3a. rows of <= SEG_MAX entries, window by window
    Buf<int32_t> ucnt(std::max<int64_t>(cn, 1), s);
    LCC_CUDA(cudaMemsetAsync(ucnt.get(), 0, sizeof(int32_t) * cn, s));
    const int64_t nwin = (nnz + SEG_WIN - 1) / SEG_WIN;
    {
        Buf<int64_t> wrow(nwin + 1, s);
        k_seg_wrow<<<grid_for(nwin + 1, 256), 256, 0, s>>>(rstart.get(), cn, nwin, wrow.get());
        LCC_LAUNCH_CHECK();
        const int SMEM = (int)sizeof(SegSmem);
        static int occ = 0;
        if (!occ) {
            LCC_CUDA(cudaFuncSetAttribute(k_seg_window, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
            LCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_seg_window, SEG_T, SMEM));
            occ = std::max(occ, 1);
        }
        const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nwin, (int64_t)num_sms() * occ));
        // (LCC_SEG_KEY64=1, tests: every window takes the 64-bit keys of windows with very many short rows)
        const int key64 = getenv("LCC_SEG_KEY64") && getenv("LCC_SEG_KEY64")[0] == '1';
        k_seg_window<<<grid, SEG_T, SMEM, s>>>(rstart.get(), wrow.get(), nwin, bbits, key64, keys.get(), vals.get(),
                                              ucnt.get());
        LCC_LAUNCH_CHECK();
    }
    tr.mark("seg windows");
    // 3b. rows of up to 8192 entries: one CTA per row (LCC_SEG_ROWS=0: the device sort takes them too)
    static const bool seg_rows_on = !(getenv("LCC_SEG_ROWS") && getenv("LCC_SEG_ROWS")[0] == '0');
    if (seg_rows_on) {
        if (SEG_MAX < 2048) seg_rows<128, 16>(rstart.get(), cn, SEG_MAX, bbits, keys.get(), vals.get(), ucnt.get(), s);
        seg_rows<256, 16>(rstart.get(), cn, std::max<int64_t>(SEG_MAX, 2048), bbits, keys.get(), vals.get(), ucnt.get(), s);
        seg_rows<512, 16>(rstart.get(), cn, 4096, bbits, keys.get(), vals.get(), ucnt.get(), s);
    }
    tr.mark("seg mid rows");
    // 3c. longer rows: one device sort of their (row, id) keys
    {
        Buf<int32_t> big(std::max<int64_t>(cn, 1), s);
        Buf<int64_t> dnb(1, s);
        select_if(cub::CountingInputIterator<int32_t>(0), big.get(), dnb.get(), cn,
                  RowLenBig{rstart.get(), seg_rows_on ? SEG_ROW_MAX : SEG_MAX}, s);
        int64_t nb = 0;
        LCC_CUDA(cudaMemcpyAsync(&nb, dnb.get(), sizeof(nb), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaStreamSynchronize(s));
        if (nb > 0) {
            Buf<int64_t> boff(nb + 1, s);
            cub::TransformInputIterator<int64_t, BigLen, cub::CountingInputIterator<int64_t>> bl(
                cub::CountingInputIterator<int64_t>(0), BigLen{rstart.get(), big.get(), nb});
            exclusive_sum(bl, boff.get(), nb + 1, s);
            int64_t bt = 0;
            LCC_CUDA(cudaMemcpyAsync(&bt, boff.get() + nb, sizeof(bt), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaStreamSynchronize(s));
            if (getenv("LCC_TRACE")) fprintf(stderr, "[lcc]     compress seg big rows: %lld rows, %lld entries\n", (long long)nb, (long long)bt);
            Buf<uint64_t> ka(bt, s), kb(bt, s);
            Buf<uint32_t> va(bt, s), vb(bt, s);
            Buf<int32_t> brank(cn, s);
            k_big_rank<<<grid_for(nb, 256), 256, 0, s>>>(big.get(), nb, brank.get());
            LCC_LAUNCH_CHECK();
            edge_balanced(rstart.get(), big.get(), boff.get(), nb, bt,
                          BigKeys{keys.get(), vals.get(), brank.get(), bbits, ka.get(), va.get()}, s);
            brank.release();
            cub::DoubleBuffer<uint64_t> dk(ka.get(), kb.get());
            cub::DoubleBuffer<uint32_t> dv(va.get(), vb.get());
            sort_pairs_db(dk, dv, bt, bbits + std::max(1, bit_width((uint64_t)std::max<int64_t>(nb - 1, 1))), s);
            Buf<uint64_t> uk(bt, s);
            Buf<uint32_t> us(bt, s);
            Buf<int64_t> druns(1, s);
            size_t bytes = 0;
            LCC_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, bytes, dk.Current(), uk.get(), dv.Current(), us.get(),
                                                    druns.get(), cub::Sum(), bt, s));
            {
                Buf<unsigned char> tmp(bytes, s);
                LCC_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), bytes, dk.Current(), uk.get(), dv.Current(),
                                                        us.get(), druns.get(), cub::Sum(), bt, s));
            }
            Buf<int64_t> first(nb, s);
            k_big_first<<<grid_for(bt, 256), 256, 0, s>>>(uk.get(), druns.get(), bbits, first.get());
            LCC_LAUNCH_CHECK();
            k_big_emit<<<grid_for(bt, 256), 256, 0, s>>>(uk.get(), us.get(), druns.get(), bbits, first.get(), big.get(),
                                                        rstart.get(), keys.get(), vals.get(), ucnt.get());
            LCC_LAUNCH_CHECK();
        }
    }
    tr.mark("seg big rows");
    // 4. exact-size coarse CSR
    cub::TransformInputIterator<int64_t, cub::CastOp<int64_t>, const int32_t*> uc(ucnt.get(), cub::CastOp<int64_t>());
    exclusive_sum(uc, out.indptr.get(), cn + 1, s);
    int64_t R = 0;
    LCC_CUDA(cudaMemcpyAsync(&R, out.indptr.get() + cn, sizeof(R), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    out.indices.alloc(std::max<int64_t>(R, 1), s);
    out.wi.alloc(std::max<int64_t>(R, 1), s);
    edge_balanced(rstart.get(), nullptr, out.indptr.get(), cn, R,
                  SegCopy{keys.get(), vals.get(), out.indices.get(), out.wi.get()}, s);
    tr.mark("seg emit");
    return R;
}

template <class WT>
Coarse compress_impl(const lcc_graph& g, const double* k, double lam, const int32_t* C, const double* K,
                     int32_t* mapping, double* ck, cudaStream_t s) {
    const int64_t n = g.n, nnz = g.nnz;
    Coarse out;
    PhaseTrace tr(s);
    const bool partial = (g.flags & LCC_GRAPH_PARTIAL_ROWS) != 0;
    // 1. dense renumbering by smallest member
    int64_t cn = 0;
    Buf<uint2> rb;  // root bitmap + sampled rank (root_rank)
    {
        Buf<int32_t> rank(n + 1, s);
        cub::TransformInputIterator<int32_t, IsRoot, cub::CountingInputIterator<int32_t>> roots(
            cub::CountingInputIterator<int32_t>(0), IsRoot{C, n});
        exclusive_sum(roots, rank.get(), n + 1, s);
        int32_t hcn = 0;
        LCC_CUDA(cudaMemcpyAsync(&hcn, rank.get() + n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        k_map<<<grid_for(n, 256), 256, 0, s>>>(C, rank.get(), K, n, mapping, ck);
        LCC_LAUNCH_CHECK();
        rb.alloc((n + 31) / 32, s);
        k_rootbits<<<grid_for((n + 31) / 32 * 32, 256), 256, 0, s>>>(C, rank.get(), n, rb.get());
        LCC_LAUNCH_CHECK();
        LCC_CUDA(cudaStreamSynchronize(s));
        cn = hcn;
    }
    out.cn = cn;
    out.indptr.alloc(cn + 1, s);
    const int bits = std::max(1, bit_width((uint64_t)cn));
    LCC_REQUIRE(2 * bits <= 64, "coarse graph too large");

    // 2. keys for every directed entry.  Integer weights (none, or uint32)
    //    stay integers: uint32 values through the sort, uint32 sums out
    //    (exact; the coarse graph is LCC_W_U32) as long as 2 * total weight
    //    fits in 32 bits; float weights carry fp64 values.
    constexpr bool FS = WLoad<WT>::fsum;
    using VT = std::conditional_t<FS, double, uint32_t>;
    const bool int_out = !FS && 2.0 * g.total_weight < 4294967296.0;
    LCC_REQUIRE((!std::is_same<WT, uint32_t>::value || int_out), "uint32 weights need 2 * total_weight < 2^32");
    out.integral = int_out;
    Buf<double> dacc(2, s);  // [intra_w, scratch]
    Buf<unsigned long long> dintra(1, s);
    LCC_CUDA(cudaMemsetAsync(dacc.get(), 0, 2 * sizeof(double), s));
    LCC_CUDA(cudaMemsetAsync(dintra.get(), 0, sizeof(unsigned long long), s));
    int64_t R = 0;
    double intra_w = 0.0;
    bool fast_done = false;
    const char* ef = getenv("LCC_CONTRACT_FAST");
    if (nnz > 0 && !(ef && ef[0] == '0')) {
        // complex rows: members of non-singleton clusters and their neighbours
        Buf<int32_t> csize(cn, s);
        LCC_CUDA(cudaMemsetAsync(csize.get(), 0, sizeof(int32_t) * cn, s));
        k_csize<<<grid_for(n, 256), 256, 0, s>>>(mapping, n, csize.get());
        LCC_LAUNCH_CHECK();
        Buf<uint8_t> cf(n, s);
        k_members<<<grid_for(n, 256), 256, 0, s>>>(mapping, csize.get(), n, cf.get());
        LCC_LAUNCH_CHECK();
        csize.release();
        Buf<int32_t> list(n, s);
        Buf<int64_t> dcount(1, s);
        auto compact_rows = [&](int64_t& cnt, Buf<int64_t>& off) {
            select_flagged(cub::CountingInputIterator<int32_t>(0), cf.get(), list.get(), dcount.get(), n, s);
            LCC_CUDA(cudaMemcpyAsync(&cnt, dcount.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaStreamSynchronize(s));
            off.alloc(cnt + 1, s);
            cub::TransformInputIterator<int64_t, DegOf, cub::CountingInputIterator<int64_t>> degs(
                cub::CountingInputIterator<int64_t>(0), DegOf{g.indptr, list.get(), cnt});
            exclusive_sum(degs, off.get(), cnt + 1, s);
            int64_t tot = 0;
            LCC_CUDA(cudaMemcpyAsync(&tot, off.get() + cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaStreamSynchronize(s));
            return tot;
        };
        int64_t nm = 0, nC = 0;
        Buf<int64_t> moff, coff;
        const int64_t mdeg = compact_rows(nm, moff);
        int64_t mc = nnz;
        if (mdeg * 10 <= nnz * 6) {  // members' rows alone already exceed the cut: full path
            if (nm > 0 && mdeg > 0)
                edge_balanced(g.indptr, list.get(), moff.get(), nm, mdeg, MarkNbrs{g.indices, cf.get()}, s);
            moff.release();
            mc = compact_rows(nC, coff);
        }
        tr.mark("classify");
        if (mc * 10 <= nnz * 6) {  // complex entries <= 60%: sort only those
            fast_done = true;
            const uint64_t sentinel = bits >= 32 ? ~0ULL : ((1ULL << (2 * bits)) - 1ULL);
            const int64_t mc1 = std::max<int64_t>(mc, 1);
            Buf<uint64_t> ka(mc1, s), kb(mc1, s);
            Buf<VT> va, vb;
            if (WLoad<WT>::weighted) { va.alloc(mc1, s); vb.alloc(mc1, s); }
            EdgeKey<WT, VT> ek{g.indices, g.weights, mapping, bits, sentinel, ka.get(), va.get(), dintra.get(),
                               dacc.get()};
            ek.compact = true;
            if (mc > 0) edge_balanced(g.indptr, list.get(), coff.get(), nC, mc, ek, s);
            cub::DoubleBuffer<uint64_t> dk(ka.get(), kb.get());
            cub::DoubleBuffer<VT> dv(va.get(), vb.get());
            if (mc > 0) {
                if (WLoad<WT>::weighted) sort_pairs_db(dk, dv, mc, 2 * bits, s);
                else sort_keys_db(dk, mc, 2 * bits, s);
            }
            Buf<uint64_t>& ksorted = dk.Current() == ka.get() ? ka : kb;
            Buf<VT>& vsorted = dv.Current() == va.get() ? va : vb;
            tr.mark("sort(cx)");
            int64_t runs = 0;
            unsigned long long hintra = 0;
            if (mc > 0) {
                Buf<int64_t> dr(1, s);
                cub::TransformInputIterator<int64_t, RunHead, cub::CountingInputIterator<int64_t>> heads(
                    cub::CountingInputIterator<int64_t>(0), RunHead{ksorted.get()});
                device_sum(heads, dr.get(), mc, s);
                LCC_CUDA(cudaMemcpyAsync(&runs, dr.get(), sizeof(runs), cudaMemcpyDeviceToHost, s));
            }
            LCC_CUDA(cudaMemcpyAsync(&hintra, dintra.get(), sizeof(hintra), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaMemcpyAsync(&intra_w, dacc.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaStreamSynchronize(s));
            const int64_t Rc = runs - (hintra > 0 ? 1 : 0);
            if (!WLoad<WT>::weighted) intra_w = (double)hintra;
            Buf<uint64_t> ukeys(std::max<int64_t>(runs, 1), s);
            Buf<uint32_t> swi;
            Buf<double> sw;
            if (int_out) swi.alloc(std::max<int64_t>(runs, 1), s);
            else sw.alloc(std::max<int64_t>(runs, 1), s);
            if (mc > 0) {
                Buf<int64_t> druns(1, s);
                auto rbk = [&](auto vals_in, auto* sums_out) {
                    size_t bytes = 0;
                    LCC_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, bytes, ksorted.get(), ukeys.get(), vals_in,
                                                            sums_out, druns.get(), cub::Sum(), mc, s));
                    Buf<unsigned char> tmp(bytes, s);
                    LCC_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), bytes, ksorted.get(), ukeys.get(), vals_in,
                                                            sums_out, druns.get(), cub::Sum(), mc, s));
                };
                if constexpr (WLoad<WT>::weighted) {
                    if constexpr (FS) rbk(vsorted.get(), sw.get());
                    else rbk(vsorted.get(), swi.get());
                } else {
                    if (int_out) rbk(cub::ConstantInputIterator<uint32_t>(1u), swi.get());
                    else rbk(cub::ConstantInputIterator<double>(1.0), sw.get());
                }
            }
            ka.release();
            kb.release();
            va.release();
            vb.release();
            tr.mark("reduce(cx)");
            // coarse row lengths -> indptr
            Buf<int64_t> clen(cn + 1, s), cstart(std::max<int64_t>(cn, 1), s);
            LCC_CUDA(cudaMemsetAsync(clen.get(), 0, sizeof(int64_t) * (cn + 1), s));
            k_simple_len<<<grid_for(n, 256), 256, 0, s>>>(g.indptr, cf.get(), mapping, n, clen.get());
            LCC_LAUNCH_CHECK();
            if (Rc > 0) {
                k_complex_start<<<grid_for(Rc, 256), 256, 0, s>>>(ukeys.get(), Rc, bits, cstart.get());
                LCC_LAUNCH_CHECK();
                k_complex_len<<<grid_for(Rc, 256), 256, 0, s>>>(ukeys.get(), Rc, bits, cstart.get(), clen.get());
                LCC_LAUNCH_CHECK();
            }
            exclusive_sum(clen.get(), out.indptr.get(), cn + 1, s);
            LCC_CUDA(cudaMemcpyAsync(&R, out.indptr.get() + cn, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaStreamSynchronize(s));
            tr.mark("lengths");
            out.indices.alloc(std::max<int64_t>(R, 1), s);
            if (int_out) out.wi.alloc(std::max<int64_t>(R, 1), s);
            else out.w.alloc(std::max<int64_t>(R, 1), s);
            tr.mark("alloc");
            if (int_out) {
                edge_balanced(g.indptr, nullptr, g.indptr, n, nnz,
                              EmitSimple<WT, uint32_t>{g.indices, g.weights, mapping, cf.get(), g.indptr,
                                                       out.indptr.get(), out.indices.get(), out.wi.get(),
                                                       partial ? nullptr : rb.get()}, s);
                if (Rc > 0) {
                    k_emit_complex<uint32_t, uint32_t><<<grid_for(Rc, 256), 256, 0, s>>>(
                        ukeys.get(), swi.get(), Rc, bits, out.indptr.get(), cstart.get(), out.indices.get(),
                        out.wi.get());
                    LCC_LAUNCH_CHECK();
                }
            } else {
                edge_balanced(g.indptr, nullptr, g.indptr, n, nnz,
                              EmitSimple<WT, double>{g.indices, g.weights, mapping, cf.get(), g.indptr,
                                                     out.indptr.get(), out.indices.get(), out.w.get(),
                                                     partial ? nullptr : rb.get()}, s);
                if (Rc > 0) {
                    k_emit_complex<double, double><<<grid_for(Rc, 256), 256, 0, s>>>(
                        ukeys.get(), sw.get(), Rc, bits, out.indptr.get(), cstart.get(), out.indices.get(),
                        out.w.get());
                    LCC_LAUNCH_CHECK();
                }
            }
            tr.mark("emit(fast)");
        }
    }
    // (when the mostly-singleton fast path did not apply) integer sums on
    // graphs of >= 2^30 entries: the segmented path, which
    // needs 8 instead of ~24-32 bytes of scratch per entry.  Measured over 6
    // config-5 clusterings (3.6B entries): 3.1-3.7 s steady state against
    // 3.6-10.4 s with the global sort, whose 60-90 GB of double-buffered keys
    // and values kept the pool re-mapping pages; config 4 (521M entries)
    // keeps the global sort and its mostly-singleton fast path (352 vs 427 ms).
    // LCC_CONTRACT_SEG=0/1 forces either.
    const char* esg = getenv("LCC_CONTRACT_SEG");
    const bool use_seg = esg ? esg[0] == '1' : nnz >= (1LL << 30);
    if (!fast_done && nnz > 0 && int_out && use_seg) {
        unsigned long long* di = dintra.get();
        // (LCC_SEG_FILLBITS=1: roots' coarse ids from the root bitmap in the fill pass; measured slower,
        // config 5 level 0: fill 96 -> 108 ms -- the test adds a dependent L2 lookup in front of every gather)
        static const bool fill_bits = getenv("LCC_SEG_FILLBITS") && getenv("LCC_SEG_FILLBITS")[0] == '1';
        R = compress_seg<WT>(g, mapping, cn, out, di, fill_bits ? rb.get() : nullptr, s);
        unsigned long long hintra = 0;
        LCC_CUDA(cudaMemcpyAsync(&hintra, di, sizeof(hintra), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaStreamSynchronize(s));
        intra_w = (double)hintra;
        fast_done = true;
        tr.mark("segmented");
    }
    if (!fast_done && nnz > 0) {
        Buf<uint64_t> ka(nnz, s), kb(nnz, s);
        Buf<VT> va, vb;
        if (WLoad<WT>::weighted) { va.alloc(nnz, s); vb.alloc(nnz, s); }
        const uint64_t sentinel = bits >= 32 ? ~0ULL : ((1ULL << (2 * bits)) - 1ULL);
        cudaEvent_t k0 = nullptr, k1 = nullptr;
        if (tr.on) { cudaEventCreate(&k0); cudaEventCreate(&k1); cudaEventRecord(k0, s); }
        edge_balanced(g.indptr, nullptr, g.indptr, n, nnz,
                      EdgeKey<WT, VT>{g.indices, g.weights, mapping, bits, sentinel, ka.get(), va.get(),
                                      dintra.get(), dacc.get()}, s);
        if (tr.on) cudaEventRecord(k1, s);
        tr.mark("keys");
        if (tr.on) {
            float kms = 0.f;
            cudaEventElapsedTime(&kms, k0, k1);
            fprintf(stderr, "[lcc]       (EdgeKey kernel alone %.2f ms)\n", kms);
            cudaEventDestroy(k0);
            cudaEventDestroy(k1);
        }
        // 3. stable radix sort on the 2*bits live bits, double-buffered (peak
        //    memory = the two key (+value) buffers, no hidden n-sized temp)
        cub::DoubleBuffer<uint64_t> dk(ka.get(), kb.get());
        cub::DoubleBuffer<VT> dv(va.get(), vb.get());
        if (WLoad<WT>::weighted) sort_pairs_db(dk, dv, nnz, 2 * bits, s);
        else sort_keys_db(dk, nnz, 2 * bits, s);
        Buf<uint64_t>& ksorted = dk.Current() == ka.get() ? ka : kb;
        (dk.Current() == ka.get() ? kb : ka).release();
        tr.mark("sort");
        Buf<VT>& vsorted = dv.Current() == va.get() ? va : vb;
        if (WLoad<WT>::weighted) (dv.Current() == va.get() ? vb : va).release();
        // 4. count the runs, then reduce by key into exact-size outputs
        //    (64-bit item counts: 2m > 2^31 at config 5)
        int64_t runs = 0;
        unsigned long long hintra = 0;
        {
            Buf<int64_t> dr(1, s);
            cub::TransformInputIterator<int64_t, RunHead, cub::CountingInputIterator<int64_t>> heads(
                cub::CountingInputIterator<int64_t>(0), RunHead{ksorted.get()});
            device_sum(heads, dr.get(), nnz, s);
            LCC_CUDA(cudaMemcpyAsync(&runs, dr.get(), sizeof(runs), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaMemcpyAsync(&hintra, dintra.get(), sizeof(hintra), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaMemcpyAsync(&intra_w, dacc.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
            LCC_CUDA(cudaStreamSynchronize(s));
        }
        R = runs - (hintra > 0 ? 1 : 0);  // the all-ones sentinel run (intra entries) sorts last
        if (!WLoad<WT>::weighted) intra_w = (double)hintra;
        Buf<uint64_t> ukeys(std::max<int64_t>(runs, 1), s);
        if (int_out) out.wi.alloc(std::max<int64_t>(runs, 1), s);
        else out.w.alloc(std::max<int64_t>(runs, 1), s);
        {
            Buf<int64_t> druns(1, s);
            auto rbk = [&](auto vals_in, auto* sums_out) {
                size_t bytes = 0;
                LCC_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, bytes, ksorted.get(), ukeys.get(), vals_in, sums_out,
                                                        druns.get(), cub::Sum(), nnz, s));
                Buf<unsigned char> tmp(bytes, s);
                LCC_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), bytes, ksorted.get(), ukeys.get(), vals_in,
                                                        sums_out, druns.get(), cub::Sum(), nnz, s));
            };
            if constexpr (WLoad<WT>::weighted) {
                if constexpr (FS) rbk(vsorted.get(), out.w.get());
                else rbk(vsorted.get(), out.wi.get());
            } else {
                if (int_out) rbk(cub::ConstantInputIterator<uint32_t>(1u), out.wi.get());
                else rbk(cub::ConstantInputIterator<double>(1.0), out.w.get());
            }
        }
        ksorted.release();
        vsorted.release();
        tr.mark("reduce");
        out.indices.alloc(std::max<int64_t>(R, 1), s);
        k_emit_rows<<<grid_for(R + 1, 256), 256, 0, s>>>(ukeys.get(), R, bits, cn, out.indptr.get(),
                                                         out.indices.get());
        LCC_LAUNCH_CHECK();
    } else if (!fast_done) {
        if (int_out) out.wi.alloc(1, s);
        else out.w.alloc(1, s);
        out.indices.alloc(1, s);
        LCC_CUDA(cudaMemsetAsync(out.indptr.get(), 0, sizeof(int64_t) * (cn + 1), s));
    }
    out.cnnz = R;
    // 5. scalars: total weight, internal offset
    Buf<double> sums(3, s);
    LCC_CUDA(cudaMemsetAsync(sums.get(), 0, 3 * sizeof(double), s));
    if (R > 0) {
        if (int_out) {
            cub::TransformInputIterator<double, U32F64, const uint32_t*> wd(out.wi.get(), U32F64{});
            device_sum(wd, sums.get() + 0, R, s);
        } else {
            device_sum(out.w.get(), sums.get() + 0, R, s);
        }
    }
    if (cn > 0) {
        cub::TransformInputIterator<double, Sq, const double*> sq(ck, Sq{});
        device_sum(sq, sums.get() + 1, cn, s);
    }
    {
        cub::TransformInputIterator<double, KSq, cub::CountingInputIterator<int64_t>> ksq(
            cub::CountingInputIterator<int64_t>(0), KSq{k});
        device_sum(ksq, sums.get() + 2, n, s);
    }
    double hs[3];
    LCC_CUDA(cudaMemcpyAsync(hs, sums.get(), sizeof(hs), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    out.total_weight = hs[0] * 0.5;
    out.internal_offset = intra_w * 0.5 - lam * (hs[1] - hs[2]) * 0.5;
    return out;
}

__global__ void k_compose(const int32_t* __restrict__ mapping, const int32_t* __restrict__ Cc, int64_t n, int32_t* D) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        D[v] = Cc[mapping[v]];
}

}  // namespace

namespace {
template <class VT>
__global__ void k_coo_keys(const int32_t* __restrict__ rows, const int32_t* __restrict__ cols,
                           const VT* __restrict__ vals, int64_t nnz, uint64_t* keys, VT* vout) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = ((uint64_t)(uint32_t)rows[i] << 32) | (uint32_t)cols[i];
        vout[i] = vals ? vals[i] : (VT)1;
    }
}
}  // namespace

// Sum duplicate (row, col) entries into a CSR: the merge step of a sharded
// contraction (partial coarse rows from several ranks; dist.py) -- the same
// key sort + run reduce as compress, with the coarse ids already assigned.
template <class VT>
int64_t coo_merge(int64_t n, int64_t nnz, const int32_t* rows, const int32_t* cols, const VT* vals,
                  int64_t* indptr, int32_t* indices, VT* wout, cudaStream_t s) {
    if (nnz <= 0) {
        LCC_CUDA(cudaMemsetAsync(indptr, 0, sizeof(int64_t) * (n + 1), s));
        return 0;
    }
    Buf<uint64_t> ka(nnz, s), kb(nnz, s);
    Buf<VT> va(nnz, s), vb(nnz, s);
    k_coo_keys<VT><<<grid_for(nnz, 256), 256, 0, s>>>(rows, cols, vals, nnz, ka.get(), va.get());
    LCC_LAUNCH_CHECK();
    cub::DoubleBuffer<uint64_t> dk(ka.get(), kb.get());
    cub::DoubleBuffer<VT> dv(va.get(), vb.get());
    sort_pairs_db(dk, dv, nnz, 32 + std::max(1, bit_width((uint64_t)std::max<int64_t>(n, 1))), s);
    Buf<uint64_t> ukeys(nnz, s);
    Buf<int64_t> druns(1, s);
    size_t bytes = 0;
    LCC_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, bytes, dk.Current(), ukeys.get(), dv.Current(), wout,
                                            druns.get(), cub::Sum(), nnz, s));
    {
        Buf<unsigned char> tmp(bytes, s);
        LCC_CUDA(cub::DeviceReduce::ReduceByKey(tmp.get(), bytes, dk.Current(), ukeys.get(), dv.Current(), wout,
                                                druns.get(), cub::Sum(), nnz, s));
    }
    int64_t R = 0;
    LCC_CUDA(cudaMemcpyAsync(&R, druns.get(), sizeof(R), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    k_emit_rows<<<grid_for(R + 1, 256), 256, 0, s>>>(ukeys.get(), R, 32, n, indptr, indices);
    LCC_LAUNCH_CHECK();
    return R;
}
template int64_t coo_merge<uint32_t>(int64_t, int64_t, const int32_t*, const int32_t*, const uint32_t*, int64_t*,
                                     int32_t*, uint32_t*, cudaStream_t);
template int64_t coo_merge<double>(int64_t, int64_t, const int32_t*, const int32_t*, const double*, int64_t*,
                                   int32_t*, double*, cudaStream_t);

Coarse compress(const lcc_graph& g, const double* k, double lam, const int32_t* C, const double* K,
                int32_t* mapping, double* ck, cudaStream_t s) {
    LCC_REQUIRE(g.n >= 0 && g.n < (1LL << 31) - 1, "vertex count out of range");
    switch (g.weights ? g.wtype : LCC_W_NONE) {
        case LCC_W_NONE: return compress_impl<WNone>(g, k, lam, C, K, mapping, ck, s);
        case LCC_W_F32: return compress_impl<float>(g, k, lam, C, K, mapping, ck, s);
        case LCC_W_F64: return compress_impl<double>(g, k, lam, C, K, mapping, ck, s);
        case LCC_W_U32: return compress_impl<uint32_t>(g, k, lam, C, K, mapping, ck, s);
        default: throw Invalid("unknown weight dtype");
    }
}

namespace {
__global__ void k_csize_c(const int32_t* __restrict__ C, int64_t n, int32_t* csize) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(csize + C[v], 1);
}
}  // namespace

// Entries the contraction of (g, C) would sort: the rows of members of
// non-singleton clusters and of their neighbours when they are at most 60% of
// nnz (the fast path of compress_impl), else nnz.  Labels must be canonical
// (< n).  Used by the driver to size the contraction before deciding to park
// finer levels on the host.
int64_t contraction_sort_entries(const lcc_graph& g, const int32_t* C, cudaStream_t s) {
    const int64_t n = g.n, nnz = g.nnz;
    if (nnz == 0 || n == 0) return 0;
    const char* ef = getenv("LCC_CONTRACT_FAST");
    if (ef && ef[0] == '0') return nnz;
    Buf<int32_t> csize(n, s);
    LCC_CUDA(cudaMemsetAsync(csize.get(), 0, sizeof(int32_t) * n, s));
    k_csize_c<<<grid_for(n, 256), 256, 0, s>>>(C, n, csize.get());
    LCC_LAUNCH_CHECK();
    Buf<uint8_t> cf(n, s);
    k_members<<<grid_for(n, 256), 256, 0, s>>>(C, csize.get(), n, cf.get());
    LCC_LAUNCH_CHECK();
    csize.release();
    Buf<int32_t> list(n, s);
    Buf<int64_t> dcount(1, s);
    auto rows = [&](int64_t& cnt, Buf<int64_t>& off) {
        select_flagged(cub::CountingInputIterator<int32_t>(0), cf.get(), list.get(), dcount.get(), n, s);
        LCC_CUDA(cudaMemcpyAsync(&cnt, dcount.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaStreamSynchronize(s));
        off.alloc(cnt + 1, s);
        cub::TransformInputIterator<int64_t, DegOf, cub::CountingInputIterator<int64_t>> degs(
            cub::CountingInputIterator<int64_t>(0), DegOf{g.indptr, list.get(), cnt});
        exclusive_sum(degs, off.get(), cnt + 1, s);
        int64_t tot = 0;
        LCC_CUDA(cudaMemcpyAsync(&tot, off.get() + cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaStreamSynchronize(s));
        return tot;
    };
    int64_t nm = 0, nc = 0;
    Buf<int64_t> moff, coff;
    const int64_t mdeg = rows(nm, moff);
    if (mdeg * 10 > nnz * 6) return nnz;
    if (nm > 0 && mdeg > 0) edge_balanced(g.indptr, list.get(), moff.get(), nm, mdeg, MarkNbrs{g.indices, cf.get()}, s);
    const int64_t mc = rows(nc, coff);
    return mc * 10 <= nnz * 6 ? mc : nnz;
}

namespace {
__global__ void k_widen_u32(const uint32_t* __restrict__ in, double* out, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}
}  // namespace

void widen_u32(const uint32_t* in, double* out, int64_t n, cudaStream_t s) {
    if (n <= 0) return;
    k_widen_u32<<<grid_for(n, 256), 256, 0, s>>>(in, out, n);
    LCC_LAUNCH_CHECK();
}

void flatten(int64_t n, const int32_t* mapping, const int32_t* Cc, const double* k, int32_t* C, double* K,
             cudaStream_t s) {
    if (n <= 0) return;
    Buf<int32_t> D(n, s);
    k_compose<<<grid_for(n, 256), 256, 0, s>>>(mapping, Cc, n, D.get());
    LCC_LAUNCH_CHECK();
    apply_moves(n, D.get(), n, k, C, K, s);
}

}  // namespace lcc
