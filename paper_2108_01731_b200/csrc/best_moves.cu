// best_moves.cu -- the best-move round (Alg. 1 lines 6-8).
//
// For every active vertex v: gather the labels of its neighbours, aggregate
// S(v,x) = sum of w(v,u) over neighbours u in cluster x, score every
// candidate with the LambdaCC gain
//     t = lambda*k_v;  b = (S_c - t*K_c) + t*k_v;  gain(x) = (S_x - t*K_x) - b
// plus the fresh-singleton option (gain -b, temporary id n+v, loses ties),
// and pick the argmax with the lowest-id tie rule; move iff gain > 0.
//
// Degree bins (all grid-stride, grids sized to the SM count):
//   small  deg <= 32   : one warp handles 32 consecutive frontier vertices,
//                        packed into 32-edge windows; labels grouped with
//                        __match_any_sync on (vertex, label); segmented
//                        argmax by warp shuffles.  Sums run in CSR order, so
//                        weighted sums are bit-identical to the oracle.
//   medium deg <= M    : one CTA per vertex, open-addressing hash table in
//                        shared memory (M set by the 227 KB/SM budget).
//   large  deg >  M    : edges split into CHUNK-edge work items spread over
//                        all SMs, inserting into a per-vertex hash table in
//                        global memory (L2-resident), then one CTA per
//                        vertex scores the table.
// sync  : targets written to D (apply happens in apply.cu);
// async : C stored and K updated with relaxed device atomics right away
//         (the CUDA analogue of _atomics.py:37-43), the
//         frontier processed in `async_chunks` ordered sub-rounds.
#include <cub/cub.cuh>
#include <math.h>
#include <type_traits>

#include "internal.cuh"
#include "prims.cuh"

namespace lcc {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int SMALL_MAX = 32;
constexpr int SMALL_THREADS = 256;
constexpr int MED_THREADS = 512;
constexpr int MED_SMEM = 110 * 1024;  // two CTAs per SM
constexpr int LARGE_CHUNK = 8192;
constexpr int LARGE_THREADS = 256;
constexpr int SCORE_THREADS = 512;

// ---- relaxed loads / stores for the async schedule ----------------------
template <bool ASYNC>
__device__ __forceinline__ int32_t ldC(const int32_t* C, int64_t i) {
    if constexpr (ASYNC) {
        int32_t r;
        asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(r) : "l"(C + i));
        return r;
    } else {
        return __ldg(C + i);
    }
}
template <bool ASYNC>
__device__ __forceinline__ double ldK(const double* K, int64_t i) {
    if constexpr (ASYNC) {
        double r;
        asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(r) : "l"(K + i));
        return r;
    } else {
        return __ldg(K + i);
    }
}
__device__ __forceinline__ void stC_relaxed(int32_t* C, int64_t i, int32_t x) {
    asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(C + i), "r"(x) : "memory");
}

struct BMArgs {
    const int64_t* indptr;
    const int32_t* indices;
    const void* w;
    const double* k;
    double lam;
    int32_t* C;
    double* K;
    int32_t* D;
    uint8_t* moved;
    unsigned long long* moved_count;
    int32_t n;
};

// Final choice for one vertex (mirrors oracle best_target()).
template <bool ASYNC>
__device__ __forceinline__ int decide(const BMArgs& a, int32_t v, int32_t c, double kv, double b,
                                      bool has, double bg, int32_t bx) {
    const double gf = dsub(0.0, b);
    int32_t choice = c;
    double cg = 0.0;
    if (has) { choice = bx; cg = bg; }
    if (!has || gf > cg) { choice = a.n + v; cg = gf; }
    if (cg > 0.0) {
        if constexpr (ASYNC) {
            stC_relaxed(a.C, v, choice);
            atomicAdd(a.K + c, -kv);
            atomicAdd(a.K + choice, kv);
        } else {
            a.D[v] = choice;
        }
        a.moved[v] = 1;
        return 1;
    }
    return 0;
}

__device__ __forceinline__ void warp_argmax(double& g, int32_t& x) {
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        double og = __shfl_xor_sync(FULL, g, d);
        int32_t ox = __shfl_xor_sync(FULL, x, d);
        if (better(og, ox, g, x)) { g = og; x = ox; }
    }
}

__device__ __forceinline__ void flush_moves(const BMArgs& a, unsigned long long mine) {
#pragma unroll
    for (int d = 16; d; d >>= 1) mine += __shfl_xor_sync(FULL, mine, d);
    if (lane_id() == 0 && mine) atomicAdd(a.moved_count, mine);
}

// ===========================================================================
// small bin: deg <= 32, warp-packed edge windows
// ===========================================================================
template <class WT, bool ASYNC>
__global__ void __launch_bounds__(SMALL_THREADS)
k_small(BMArgs a, const int32_t* __restrict__ list, int64_t lo, int64_t hi) {
    constexpr int WPB = SMALL_THREADS / 32;
    __shared__ int32_t s_owner[WPB][32];
    __shared__ double s_sc[WPB][32];
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nb = (hi - lo + 31) / 32;
    const int64_t gw = ((int64_t)blockIdx.x * SMALL_THREADS + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * SMALL_THREADS) >> 5;
    unsigned long long my_moves = 0;

    for (int64_t bt = gw; bt < nb; bt += nw) {
        const int64_t i0 = lo + bt * 32;
        const int nvalid = (int)min64(32, hi - i0);
        const bool valid = lane < nvalid;
        int32_t v = 0, deg = 0, c = 0;
        int64_t s = 0;
        double kv = 1.0, Kc = 0.0;
        if (valid) {
            v = __ldg(list + i0 + lane);
            s = __ldg(a.indptr + v);
            deg = (int32_t)(__ldg(a.indptr + v + 1) - s);
            c = ldC<ASYNC>(a.C, v);
            kv = kval(a.k, v);
            Kc = ldK<ASYNC>(a.K, c);
        }
        const double t = dmul(a.lam, kv);
        int32_t incl = deg;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int32_t y = __shfl_up_sync(FULL, incl, d);
            if (lane >= d) incl += y;
        }
        const int32_t excl = incl - deg;

        int base = 0;
        while (base < nvalid) {
            const int32_t base_off = __shfl_sync(FULL, excl, base);
            const bool inwin = valid && lane >= base && (incl - base_off) <= SMALL_MAX;
            const unsigned winmask = __ballot_sync(FULL, inwin);
            const int end = 32 - __clz(winmask);
            const int32_t nedges = __shfl_sync(FULL, incl, end - 1) - base_off;
            const int32_t rs = excl - base_off;
            const bool starter = inwin && deg > 0;
            const unsigned starts = __reduce_or_sync(FULL, starter ? (1u << rs) : 0u);
            if (starter) s_owner[wib][rs] = lane;
            if (inwin) s_sc[wib][lane] = 0.0;
            __syncwarp();

            const bool has_edge = lane < nedges;
            int p = 0, j = 0;
            if (has_edge) {
                const unsigned m = starts & ((2u << lane) - 1u);
                p = 31 - __clz(m);
                j = s_owner[wib][p];
            }
            const int64_t sj = __shfl_sync(FULL, s, j);
            const int32_t cj = __shfl_sync(FULL, c, j);
            const double tj = __shfl_sync(FULL, t, j);
            int32_t x = 0;
            double wv = 0.0;
            if (has_edge) {
                const int64_t e = sj + (lane - p);
                x = ldC<ASYNC>(a.C, __ldg(a.indices + e));
                wv = WLoad<WT>::at(a.w, e);
            }
            const uint64_t key = has_edge ? (((uint64_t)(uint32_t)j << 32) | (uint32_t)x)
                                          : ((uint64_t)(64 + lane) << 32);
            const unsigned grp = __match_any_sync(FULL, key);
            double S;
            if constexpr (!WLoad<WT>::weighted) {
                S = (double)__popc(grp);
            } else {
                S = 0.0;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const double wq = __shfl_sync(FULL, wv, q);
                    if ((grp >> q) & 1u) S = dadd(S, wq);
                }
            }
            const bool is_leader = has_edge && lane == (__ffs(grp) - 1);
            if (is_leader && x == cj) s_sc[wib][j] = S;
            __syncwarp();
            double bv = 0.0;
            if (inwin) bv = dadd(dsub(s_sc[wib][lane], dmul(t, Kc)), dmul(t, kv));
            const double bj = __shfl_sync(FULL, bv, j);
            double g = -INFINITY;
            int32_t gx = NO_CAND;
            if (is_leader && x != cj) {
                g = dsub(dsub(S, dmul(tj, ldK<ASYNC>(a.K, x))), bj);
                gx = x;
            }
            const int32_t seg = has_edge ? j : 32 + lane;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double og = __shfl_down_sync(FULL, g, d);
                const int32_t ox = __shfl_down_sync(FULL, gx, d);
                const int32_t os = __shfl_down_sync(FULL, seg, d);
                if (lane + d < 32 && os == seg && better(og, ox, g, gx)) { g = og; gx = ox; }
            }
            const int src = starter ? rs : lane;
            const double hg = __shfl_sync(FULL, g, src);
            const int32_t hx = __shfl_sync(FULL, gx, src);
            if (inwin) my_moves += decide<ASYNC>(a, v, c, kv, bv, starter && hx != NO_CAND, hg, hx);
            base = end;
            __syncwarp();
        }
    }
    flush_moves(a, my_moves);
}

// ===========================================================================
// shared hash-table helpers (medium bin: smem, large bin: global)
// ===========================================================================
__device__ __forceinline__ uint32_t slot_of(int32_t x, uint32_t cap) {
    return (uint32_t)(((uint64_t)hash32((uint32_t)x) * cap) >> 32);
}

template <class VT>
__device__ __forceinline__ void table_insert(int32_t* keys, VT* vals, uint32_t cap, int32_t x, double wv) {
    uint32_t h = slot_of(x, cap);
    volatile int32_t* vk = keys;
    while (true) {
        const int32_t kq = vk[h];
        if (kq == x) break;
        if (kq == EMPTY_KEY) {
            const int32_t prev = atomicCAS(keys + h, EMPTY_KEY, x);
            if (prev == EMPTY_KEY || prev == x) break;
        }
        h = (h + 1 == cap) ? 0 : h + 1;
    }
    if constexpr (std::is_same<VT, double>::value) atomicAdd(vals + h, wv);
    else atomicAdd(vals + h, (VT)1);
}

template <class VT>
__device__ __forceinline__ double table_lookup(const int32_t* keys, const VT* vals, uint32_t cap, int32_t x) {
    uint32_t h = slot_of(x, cap);
    for (uint32_t probes = 0; probes < cap; ++probes) {
        const int32_t kq = keys[h];
        if (kq == x) return (double)vals[h];
        if (kq == EMPTY_KEY) return 0.0;
        h = (h + 1 == cap) ? 0 : h + 1;
    }
    return 0.0;
}

template <int THREADS>
__device__ __forceinline__ void block_argmax(double& g, int32_t& x, double* s_g, int32_t* s_x) {
    warp_argmax(g, x);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { s_g[w] = g; s_x[w] = x; }
    __syncthreads();
    if (threadIdx.x < 32) {
        g = threadIdx.x < THREADS / 32 ? s_g[threadIdx.x] : -INFINITY;
        x = threadIdx.x < THREADS / 32 ? s_x[threadIdx.x] : NO_CAND;
        warp_argmax(g, x);
    }
}

template <class WT>
using ValT = typename std::conditional<WLoad<WT>::weighted, double, int32_t>::type;

template <class WT>
constexpr int med_capacity() {
    return (MED_SMEM - 64) / (int)(sizeof(int32_t) + sizeof(ValT<WT>));
}

// ===========================================================================
// medium bin: one CTA per vertex, shared-memory hash table
// ===========================================================================
template <class WT, bool ASYNC>
__global__ void __launch_bounds__(MED_THREADS, 2)
k_medium(BMArgs a, const int32_t* __restrict__ list, int64_t lo, int64_t hi) {
    using VT = ValT<WT>;
    constexpr int CAP = med_capacity<WT>();
    extern __shared__ __align__(16) unsigned char smem[];
    VT* vals = reinterpret_cast<VT*>(smem);
    int32_t* keys = reinterpret_cast<int32_t*>(vals + CAP);
    __shared__ double s_g[MED_THREADS / 32];
    __shared__ int32_t s_x[MED_THREADS / 32];
    __shared__ double s_sc;
    unsigned long long my_moves = 0;

    for (int64_t i = lo + blockIdx.x; i < hi; i += gridDim.x) {
        const int32_t v = __ldg(list + i);
        const int64_t s = __ldg(a.indptr + v);
        const int64_t deg = __ldg(a.indptr + v + 1) - s;
        const uint32_t cap = (uint32_t)min64(CAP, (2 * deg + 31) & ~31LL);
        for (uint32_t q = threadIdx.x; q < cap; q += MED_THREADS) { keys[q] = EMPTY_KEY; vals[q] = (VT)0; }
        const int32_t c = ldC<ASYNC>(a.C, v);
        const double kv = kval(a.k, v);
        const double Kc = ldK<ASYNC>(a.K, c);
        const double t = dmul(a.lam, kv);
        __syncthreads();
        for (int64_t e = s + threadIdx.x; e < s + deg; e += MED_THREADS) {
            const int32_t x = ldC<ASYNC>(a.C, __ldg(a.indices + e));
            table_insert<VT>(keys, vals, cap, x, WLoad<WT>::at(a.w, e));
        }
        __syncthreads();
        if (threadIdx.x == 0) s_sc = table_lookup<VT>(keys, vals, cap, c);
        __syncthreads();
        const double b = dadd(dsub(s_sc, dmul(t, Kc)), dmul(t, kv));
        double bg = -INFINITY;
        int32_t bx = NO_CAND;
        for (uint32_t q = threadIdx.x; q < cap; q += MED_THREADS) {
            const int32_t x = keys[q];
            if (x != EMPTY_KEY && x != c) {
                const double gq = dsub(dsub((double)vals[q], dmul(t, ldK<ASYNC>(a.K, x))), b);
                if (better(gq, x, bg, bx)) { bg = gq; bx = x; }
            }
        }
        block_argmax<MED_THREADS>(bg, bx, s_g, s_x);
        if (threadIdx.x == 0) my_moves += decide<ASYNC>(a, v, c, kv, b, bx != NO_CAND, bg, bx);
        __syncthreads();
    }
    if (threadIdx.x < 32) flush_moves(a, my_moves);
}

// ===========================================================================
// large bin: multi-CTA insertion into global hash tables, CTA-per-vertex scoring
// ===========================================================================
struct LargeLayout {
    const int32_t* list;     // large-bin vertices
    int64_t nL;
    const int64_t* cap_off;  // [nL+1] table offsets
    const int64_t* item_off; // [nL+1] work-item offsets
    int32_t* keys;
    void* vals;
};

__global__ void k_large_sizes(const int64_t* __restrict__ indptr, const int32_t* __restrict__ list,
                              int64_t nL, int64_t* caps, int64_t* items) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= nL; i += (int64_t)gridDim.x * blockDim.x) {
        if (i == nL) { caps[i] = 0; items[i] = 0; continue; }
        const int32_t v = list[i];
        const int64_t deg = indptr[v + 1] - indptr[v];
        caps[i] = (2 * deg + 31) & ~31LL;
        items[i] = (deg + LARGE_CHUNK - 1) / LARGE_CHUNK;
    }
}

template <class WT, bool ASYNC>
__global__ void __launch_bounds__(LARGE_THREADS)
k_large_insert(BMArgs a, LargeLayout L, int64_t total_items) {
    using VT = ValT<WT>;
    for (int64_t it = blockIdx.x; it < total_items; it += gridDim.x) {
        // owner: last li with item_off[li] <= it
        int64_t lo = 0, hi = L.nL;  // item_off[0] = 0 <= it < item_off[nL]
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (L.item_off[mid] <= it) lo = mid; else hi = mid;
        }
        const int32_t v = L.list[lo];
        const int64_t s = a.indptr[v], e_end = a.indptr[v + 1];
        const int64_t e0 = s + (it - L.item_off[lo]) * LARGE_CHUNK;
        const int64_t e1 = min64(e0 + LARGE_CHUNK, e_end);
        const uint32_t cap = (uint32_t)(L.cap_off[lo + 1] - L.cap_off[lo]);
        int32_t* keys = L.keys + L.cap_off[lo];
        VT* vals = static_cast<VT*>(L.vals) + L.cap_off[lo];
        for (int64_t e = e0 + threadIdx.x; e < e1; e += LARGE_THREADS) {
            const int32_t x = ldC<ASYNC>(a.C, __ldg(a.indices + e));
            table_insert<VT>(keys, vals, cap, x, WLoad<WT>::at(a.w, e));
        }
    }
}

template <class WT, bool ASYNC>
__global__ void __launch_bounds__(SCORE_THREADS)
k_large_score(BMArgs a, LargeLayout L) {
    using VT = ValT<WT>;
    __shared__ double s_g[SCORE_THREADS / 32];
    __shared__ int32_t s_x[SCORE_THREADS / 32];
    __shared__ double s_sc;
    unsigned long long my_moves = 0;
    for (int64_t li = blockIdx.x; li < L.nL; li += gridDim.x) {
        const int32_t v = L.list[li];
        const uint32_t cap = (uint32_t)(L.cap_off[li + 1] - L.cap_off[li]);
        const int32_t* keys = L.keys + L.cap_off[li];
        const VT* vals = static_cast<const VT*>(L.vals) + L.cap_off[li];
        const int32_t c = ldC<ASYNC>(a.C, v);
        const double kv = kval(a.k, v);
        const double Kc = ldK<ASYNC>(a.K, c);
        const double t = dmul(a.lam, kv);
        if (threadIdx.x == 0) s_sc = table_lookup<VT>(keys, vals, cap, c);
        __syncthreads();
        const double b = dadd(dsub(s_sc, dmul(t, Kc)), dmul(t, kv));
        double bg = -INFINITY;
        int32_t bx = NO_CAND;
        for (uint32_t q = threadIdx.x; q < cap; q += SCORE_THREADS) {
            const int32_t x = keys[q];
            if (x != EMPTY_KEY && x != c) {
                const double gq = dsub(dsub((double)vals[q], dmul(t, ldK<ASYNC>(a.K, x))), b);
                if (better(gq, x, bg, bx)) { bg = gq; bx = x; }
            }
        }
        block_argmax<SCORE_THREADS>(bg, bx, s_g, s_x);
        if (threadIdx.x == 0) my_moves += decide<ASYNC>(a, v, c, kv, b, bx != NO_CAND, bg, bx);
        __syncthreads();
    }
    if (threadIdx.x < 32) flush_moves(a, my_moves);
}

// ---- degree predicates for the bin partition -----------------------------
struct DegBetween {
    const int64_t* indptr;
    int64_t lo, hi;  // lo < deg <= hi
    __device__ __forceinline__ bool operator()(int32_t v) const {
        const int64_t d = indptr[v + 1] - indptr[v];
        return d > lo && d <= hi;
    }
};
struct DegOf {
    const int64_t* indptr;
    __device__ __forceinline__ int64_t operator()(int32_t v) const { return indptr[v + 1] - indptr[v]; }
};

template <class It>
void partition_bins(It in, int64_t nF, const int64_t* indptr, int64_t med_max, int32_t* small,
                    int32_t* med, int32_t* large, int64_t* d_counts, cudaStream_t s) {
    select_if(in, small, d_counts + 0, nF, DegBetween{indptr, -1, SMALL_MAX}, s);
    select_if(in, med, d_counts + 1, nF, DegBetween{indptr, SMALL_MAX, med_max}, s);
    select_if(in, large, d_counts + 2, nF, DegBetween{indptr, med_max, INT64_MAX}, s);
    cub::TransformInputIterator<int64_t, DegOf, It> degs(in, DegOf{indptr});
    device_sum(degs, d_counts + 3, nF, s);
}

template <class WT, bool ASYNC>
void set_smem_attr() {
    static bool done = false;
    if (!done) {
        LCC_CUDA(cudaFuncSetAttribute(k_medium<WT, ASYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, MED_SMEM));
        done = true;
    }
}

template <class WT, bool ASYNC>
int64_t run_round(const lcc_graph& g, const double* k, double lam, int32_t* C, double* K,
                  const int32_t* frontier, int64_t nF, int deg_threshold, int chunks, int32_t* D,
                  uint8_t* moved, RoundStats* st, cudaStream_t s) {
    const int64_t n = g.n;
    constexpr int64_t CAP = med_capacity<WT>();
    const int64_t med_max = std::max<int64_t>((int64_t)deg_threshold, (CAP * 2) / 3);
    if (!ASYNC) LCC_CUDA(cudaMemcpyAsync(D, C, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
    LCC_CUDA(cudaMemsetAsync(moved, 0, n, s));

    Buf<int32_t> lists(3 * (size_t)std::max<int64_t>(nF, 1), s);
    int32_t* small = lists.get();
    int32_t* med = small + nF;
    int32_t* large = med + nF;
    Buf<int64_t> dcnt(4, s);
    Buf<unsigned long long> dmoved(1, s);
    LCC_CUDA(cudaMemsetAsync(dmoved.get(), 0, sizeof(unsigned long long), s));
    if (frontier) partition_bins(frontier, nF, g.indptr, med_max, small, med, large, dcnt.get(), s);
    else partition_bins(cub::CountingInputIterator<int32_t>(0), nF, g.indptr, med_max, small, med, large, dcnt.get(), s);
    int64_t hc[4];
    LCC_CUDA(cudaMemcpyAsync(hc, dcnt.get(), sizeof(hc), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    const int64_t nS = hc[0], nM = hc[1], nL = hc[2];

    BMArgs a{g.indptr, g.indices, g.weights, k, lam, C, K, D, moved, dmoved.get(), (int32_t)n};
    set_smem_attr<WT, ASYNC>();
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    LCC_CUDA(cudaEventCreate(&ev0));
    LCC_CUDA(cudaEventCreate(&ev1));
    const long long launches0 = launch_counter();
    float kms = 0.f, kms_large = 0.f;

    // large bin: one pass over all large vertices (first sub-round)
    Buf<int64_t> lbuf;
    Buf<int32_t> lkeys;
    Buf<unsigned char> lvals;
    if (nL > 0) {
        lbuf.alloc(2 * (nL + 1) * 2, s);
        int64_t* caps = lbuf.get();
        int64_t* items = caps + (nL + 1);
        int64_t* cap_off = items + (nL + 1);
        int64_t* item_off = cap_off + (nL + 1);
        k_large_sizes<<<grid_for(nL + 1, 256), 256, 0, s>>>(g.indptr, large, nL, caps, items);
        LCC_LAUNCH_CHECK();
        exclusive_sum(caps, cap_off, nL + 1, s);
        exclusive_sum(items, item_off, nL + 1, s);
        int64_t tot[2];
        LCC_CUDA(cudaMemcpyAsync(&tot[0], cap_off + nL, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaMemcpyAsync(&tot[1], item_off + nL, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaStreamSynchronize(s));
        lkeys.alloc(tot[0], s);
        lvals.alloc(tot[0] * sizeof(ValT<WT>), s);
        LCC_CUDA(cudaMemsetAsync(lkeys.get(), 0xff, sizeof(int32_t) * tot[0], s));
        LCC_CUDA(cudaMemsetAsync(lvals.get(), 0, sizeof(ValT<WT>) * tot[0], s));
        LargeLayout L{large, nL, cap_off, item_off, lkeys.get(), lvals.get()};
        LCC_CUDA(cudaEventRecord(ev0, s));
        k_large_insert<WT, ASYNC><<<grid_for(tot[1] * LARGE_THREADS, LARGE_THREADS, 16), LARGE_THREADS, 0, s>>>(a, L, tot[1]);
        LCC_LAUNCH_CHECK();
        k_large_score<WT, ASYNC><<<grid_for(nL * SCORE_THREADS, SCORE_THREADS, 4), SCORE_THREADS, 0, s>>>(a, L);
        LCC_LAUNCH_CHECK();
        LCC_CUDA(cudaEventRecord(ev1, s));
        LCC_CUDA(cudaEventSynchronize(ev1));
        LCC_CUDA(cudaEventElapsedTime(&kms_large, ev0, ev1));
    }
    const int P = ASYNC ? std::max(1, chunks) : 1;
    LCC_CUDA(cudaEventRecord(ev0, s));
    for (int j = 0; j < P; ++j) {
        const int64_t s0 = nS * j / P, s1 = nS * (j + 1) / P;
        const int64_t m0 = nM * j / P, m1 = nM * (j + 1) / P;
        if (s1 > s0) {
            const int64_t warps = (s1 - s0 + 31) / 32;
            k_small<WT, ASYNC><<<grid_for(warps * 32, SMALL_THREADS, 8), SMALL_THREADS, 0, s>>>(a, small, s0, s1);
            LCC_LAUNCH_CHECK();
        }
        if (m1 > m0) {
            k_medium<WT, ASYNC><<<grid_for((m1 - m0) * MED_THREADS, MED_THREADS, 2), MED_THREADS, MED_SMEM, s>>>(a, med, m0, m1);
            LCC_LAUNCH_CHECK();
        }
    }
    LCC_CUDA(cudaEventRecord(ev1, s));
    unsigned long long hm = 0;
    LCC_CUDA(cudaMemcpyAsync(&hm, dmoved.get(), sizeof(hm), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    LCC_CUDA(cudaEventElapsedTime(&kms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    if (st) {
        st->vertices += nF;
        st->edges += hc[3];
        st->moved += (int64_t)hm;
        st->n_small += nS;
        st->n_medium += nM;
        st->n_large += nL;
        st->ms_kernels += (double)kms + (double)kms_large;
        st->launches += launch_counter() - launches0;
    }
    return (int64_t)hm;
}

}  // namespace

int64_t best_moves_round(const lcc_graph& g, const double* k, double lam, int32_t* C, double* K,
                         const int32_t* frontier, int64_t nF, int schedule, int deg_threshold,
                         int async_chunks, int32_t* D, uint8_t* moved, RoundStats* st,
                         cudaStream_t s) {
    LCC_REQUIRE(g.n >= 0 && g.n < (1LL << 30), "vertex count out of range");
    LCC_REQUIRE(schedule == LCC_SYNC || schedule == LCC_ASYNC, "unknown schedule");
    LCC_REQUIRE(schedule == LCC_ASYNC || D != nullptr, "sync schedule needs D");
    if (!frontier) nF = g.n;
    if (g.n == 0) return 0;
    const bool as = schedule == LCC_ASYNC;
    switch (g.weights ? g.wtype : LCC_W_NONE) {
        case LCC_W_NONE:
            return as ? run_round<WNone, true>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, st, s)
                      : run_round<WNone, false>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, st, s);
        case LCC_W_F32:
            return as ? run_round<float, true>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, st, s)
                      : run_round<float, false>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, st, s);
        case LCC_W_F64:
            return as ? run_round<double, true>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, st, s)
                      : run_round<double, false>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, st, s);
        default:
            throw Invalid("unknown weight dtype");
    }
}

}  // namespace lcc
