// edgemap.cuh -- edge-balanced traversal of a vertex list's adjacency.
//
// Work is split into fixed tiles of the concatenated edge space, so a
// 400K-degree hub costs the same per edge as a degree-3 vertex (a warp- or
// block-per-vertex mapping leaves a single warp walking the hub).  For each
// edge position e the owning list entry is found by a binary search of the
// degree prefix `off` restricted to the tile's window (found once per tile).
// `off` is the exclusive degree prefix over `list` (off[nlist] = total); for
// the all-vertices case pass list = nullptr and off = indptr.
#pragma once
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace lcc {

constexpr int EM_THREADS = 256;
constexpr int EM_ITEMS = 8;
constexpr int EM_TILE = EM_THREADS * EM_ITEMS;

__device__ __forceinline__ int64_t upper_idx(const int64_t* off, int64_t lo, int64_t hi, int64_t e) {
    // largest a in [lo, hi) with off[a] <= e, given off[lo] <= e
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(off + mid) <= e) lo = mid; else hi = mid;
    }
    return lo;
}

// F: functor with  __device__ void operator()(int64_t v, int64_t e, int64_t pos)
//    (v = list entry's vertex, e = its CSR edge index, pos = position in the
//    concatenated edge space [0, off[nlist]))  and
//                  __device__ void flush()   (called once per thread at the end)
// When the tile's window of `off` fits in shared memory (always the case for
// lists whose entries all have degree >= 1: at most EM_TILE + 1 entries) the
// per-edge search runs in shared memory; otherwise it falls back to global.
// first and one-past-last list entry owning each tile, found for all tiles at
// once (a tile that searched for itself spent ~25 dependent global loads
// before its first edge: config-5 fast-path emit 49 -> 39 ms, segmented emit 40 -> 28 ms with this)
static __global__ void k_tile_bounds(const int64_t* __restrict__ off, int64_t nlist, int64_t tiles, int64_t* __restrict__ tlo,
                              int64_t* __restrict__ thi) {
    const int64_t total = __ldg(off + nlist);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tiles; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t0 = t * EM_TILE, t1 = min64(t0 + EM_TILE, total);
        tlo[t] = upper_idx(off, 0, nlist + 1, t0);
        thi[t] = upper_idx(off, 0, nlist + 1, t1 - 1) + 1;
    }
}

// Two-phase functors (a nested `Tmp` type, `Tmp load(v, e, pos)` and
// `void store(const Tmp&, v, e, pos)`): all EM_ITEMS loads of a thread are
// issued before its first store.  With a plain operator() the compiler must
// keep every element's loads behind the previous element's stores (the
// output may alias the input for all it knows), which serialised 8 load ->
// store round trips per thread and tile: the emit copy of the segmented
// contraction ran at 1.7 TB/s with 66% of its stall samples on those loads
// (profiles/s6_contract_ncu.md).
template <class F, class = void>
struct em_two_phase : std::false_type {};
template <class F>
struct em_two_phase<F, std::void_t<typename F::Tmp>> : std::true_type {};

// Functors with `int64_t prep(int64_t v)`: evaluated once per list entry of a
// tile (shared memory), and load()/store() receive that value in place of v --
// the per-row part of an address (a flag, a mapping and two row offsets for the
// fast-path emit) is not re-read for every entry of the row.
template <class F, class = void>
struct em_has_prep : std::false_type {};
template <class F>
struct em_has_prep<F, std::void_t<decltype(&F::prep)>> : std::true_type {};

template <class F>
__global__ void __launch_bounds__(EM_THREADS)
k_edge_balanced(const int64_t* __restrict__ indptr, const int32_t* __restrict__ list,
                const int64_t* __restrict__ off, int64_t nlist, const int64_t* __restrict__ tlo,
                const int64_t* __restrict__ thi, F f) {
    __shared__ int32_t s_off[EM_TILE + 2];  // entry starts relative to the tile, clamped to [-1, EM_TILE + 1]
    __shared__ int64_t s_row[EM_TILE + 1];  // start of each window entry's row
    __shared__ int32_t s_v[em_has_prep<F>::value ? 1 : EM_TILE + 1];  // vertex of each window entry
    constexpr bool PREP = em_has_prep<F>::value;
    static_assert(!PREP || em_two_phase<F>::value, "prep() goes with load()/store()");
    __shared__ int64_t s_aux[PREP ? EM_TILE + 1 : 1];  // f.prep(vertex)
    const int64_t total = __ldg(off + nlist);
    for (int64_t t0 = (int64_t)blockIdx.x * EM_TILE; t0 < total; t0 += (int64_t)gridDim.x * EM_TILE) {
        const int64_t t1 = min64(t0 + EM_TILE, total);
        const int64_t lo = __ldg(tlo + t0 / EM_TILE), hi = __ldg(thi + t0 / EM_TILE);
        const int64_t wn = hi - lo;  // entries lo .. hi-1 own the tile; off[hi] closes it
        const bool cached = wn <= EM_TILE;
        if (cached) {
            for (int64_t i = threadIdx.x; i <= wn; i += EM_THREADS) {
                const int64_t r = __ldg(off + lo + i) - t0;
                s_off[i] = (int32_t)(r < -1 ? -1 : (r > EM_TILE + 1 ? EM_TILE + 1 : r));
            }
            for (int64_t i = threadIdx.x; i < wn; i += EM_THREADS) {
                const int64_t v = list ? (int64_t)__ldg(list + lo + i) : lo + i;
                if constexpr (!PREP) s_v[i] = (int32_t)v;
                s_row[i] = __ldg(indptr + v) - __ldg(off + lo + i);  // edge e of this entry = s_row + e
                if constexpr (PREP) s_aux[i] = f.prep(v);
            }
        }
        __syncthreads();
        if (cached) {
            // owners of all EM_ITEMS positions first (shared-memory searches),
            // then the functor calls as straight-line code, so their global
            // gathers are all in flight together
            int own[EM_ITEMS];
#pragma unroll
            for (int j = 0; j < EM_ITEMS; ++j) {
                const int64_t e = t0 + (int64_t)j * EM_THREADS + threadIdx.x;
                int a = 0, b = (int)wn;  // largest a with s_off[a] <= e
                if (e < t1) {
                    while (b - a > 1) {
                        const int mid = (a + b) >> 1;
                        if (s_off[mid] <= (int32_t)(e - t0)) a = mid; else b = mid;
                    }
                }
                own[j] = a;
            }
            if constexpr (em_two_phase<F>::value) {
                typename F::Tmp tmp[EM_ITEMS];
#pragma unroll
                for (int j = 0; j < EM_ITEMS; ++j) {
                    const int64_t e = t0 + (int64_t)j * EM_THREADS + threadIdx.x;
                    if (e < t1) tmp[j] = f.load(PREP ? s_aux[own[j]] : (int64_t)s_v[PREP ? 0 : own[j]], s_row[own[j]] + e, e);
                }
#pragma unroll
                for (int j = 0; j < EM_ITEMS; ++j) {
                    const int64_t e = t0 + (int64_t)j * EM_THREADS + threadIdx.x;
                    if (e < t1) f.store(tmp[j], PREP ? s_aux[own[j]] : (int64_t)s_v[PREP ? 0 : own[j]], s_row[own[j]] + e, e);
                }
            } else {
#pragma unroll
                for (int j = 0; j < EM_ITEMS; ++j) {
                    const int64_t e = t0 + (int64_t)j * EM_THREADS + threadIdx.x;
                    if (e < t1) f((int64_t)s_v[own[j]], s_row[own[j]] + e, e);
                }
            }
        } else {
#pragma unroll 2
            for (int j = 0; j < EM_ITEMS; ++j) {
                const int64_t e = t0 + (int64_t)j * EM_THREADS + threadIdx.x;
                if (e < t1) {
                    const int64_t li = upper_idx(off, lo, hi, e);
                    const int64_t v = list ? (int64_t)__ldg(list + li) : li;
                    const int64_t ee = __ldg(indptr + v) + (e - __ldg(off + li));
                    if constexpr (PREP) {
                        const int64_t ax = f.prep(v);
                        f.store(f.load(ax, ee, e), ax, ee, e);
                    } else if constexpr (em_two_phase<F>::value) f.store(f.load(v, ee, e), v, ee, e);
                    else f(v, ee, e);
                }
            }
        }
        __syncthreads();
    }
    f.flush();
}

template <class F>
inline void edge_balanced(const int64_t* indptr, const int32_t* list, const int64_t* off, int64_t nlist,
                          int64_t total_edges, F f, cudaStream_t s) {
    if (total_edges <= 0) return;
    const int64_t tiles = (total_edges + EM_TILE - 1) / EM_TILE;
    const int64_t cap = (int64_t)num_sms() * 8;
    const unsigned grid = (unsigned)(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
    Buf<int64_t> tlo(tiles, s), thi(tiles, s);
    k_tile_bounds<<<(unsigned)std::min<int64_t>((tiles + 255) / 256, 65535), 256, 0, s>>>(off, nlist, tiles, tlo.get(),
                                                                                         thi.get());
    LCC_LAUNCH_CHECK();
    k_edge_balanced<F><<<grid, EM_THREADS, 0, s>>>(indptr, list, off, nlist, tlo.get(), thi.get(), f);
    LCC_LAUNCH_CHECK();
}

}  // namespace lcc
