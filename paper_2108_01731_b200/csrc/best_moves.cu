// best_moves.cu -- the best-move round (Alg. 1 lines 6-8).
//
// For every active vertex v: gather the labels of its neighbours, aggregate
// S(v,x) = sum of w(v,u) over neighbours u in cluster x, score every
// candidate with the LambdaCC gain
//     t = lambda*k_v;  b = (S_c - t*K_c) + t*k_v;  gain(x) = (S_x - t*K_x) - b
// plus the fresh-singleton option (gain -b, temporary id n+v, loses ties),
// and pick the argmax with the lowest-id tie rule; move iff gain > 0.
//
// The frontier is split by degree into bins (stable two-pass partition),
// each with a kernel whose thread count matches the work:
//   0  isolated            : k_isolated, thread per vertex (fresh singleton only)
//   1  deg <= 8            : k_tiny, thread per vertex, labels in registers
//   2  deg <= 32           : k_small, one warp packs 32 vertices into 32-edge
//                            windows; labels grouped by __match_any_sync on
//                            (vertex, label); segmented argmax by shuffles.
//                            Sums run in CSR order (bit-identical to the oracle
//                            even for weighted graphs).
//   3  (opt-in LCC_WINDOW) : k_window, edge-balanced multi-vertex CTAs
//   4-5 33 .. 512          : k_group, one WARP per vertex, 256/1024-slot
//                            shared-memory hash table (the paper's
//                            "sequential" per-vertex accumulation)
//   6-9 .. 10240           : k_group, 4/4/8/32 warps per vertex, 2K-16K slots
//                            ("parallel hash table")
//   10 hubs                : labels radix-partitioned by hash into ~2K-entry
//                            buckets, each aggregated by one CTA in a 4K-slot
//                            shared-memory table (k_hub_*); LCC_HUB_BUCKETS=0:
//                            2048-edge items inserting into per-vertex global
//                            (L2) tables; opt-in DSMEM cluster tables
//                            (LCC_HUB_CLUSTER=1).
// Tables use native 32-bit shared atomics (CAS on the key, RED on the
// count / integer weight); float weights add with fp64 RED.
// sync  : targets written to D (apply happens in apply.cu);
// async : C stored and K updated with relaxed device atomics right away
//         (the CUDA analogue of _atomics.py:37-43), the
//         frontier processed in ordered sub-rounds for small frontiers, and
//         every move re-validated at commit time against the target's mass
//         returned by the join atomic (no stale-mass pile-ups).
// Optional fused VertexNeighbors frontier: movers flag their neighbours.
#include <cub/cub.cuh>
#include <math.h>
#include <type_traits>
#include <vector>
#include <cstdlib>
#include <chrono>
#include <thread>
#include <cstdio>

#include "internal.cuh"
#include "prims.cuh"

namespace lcc {
namespace {

#ifndef LCC_FHASH
#define LCC_FHASH 1  // Fibonacci slot hash (+0.8% vs the murmur finalizer)
#endif
#ifndef LCC_LDS_FIRST
#define LCC_LDS_FIRST 0  // 1: read the slot before the atomic (measured 28% slower: a dependent LDS per probe)
#endif
#ifndef LCC_ALWAYS_RED
#define LCC_ALWAYS_RED 0  // tuning: RED even for unit-weight claims
#endif
#ifndef LCC_SMALL_PIPE
#define LCC_SMALL_PIPE 1  // k_small: next window's loads issued before this window is processed
#endif
#ifndef LCC_SMALL_LADDER2
#define LCC_SMALL_LADDER2 1  // k_small: segment bounds from the starts mask, S fetched after the ladder
#endif
#ifndef LCC_VALIDATE
#define LCC_VALIDATE 1  // async: re-check the gain with the target's mass at commit time
#endif
#ifndef LCC_TMAPF
#define LCC_TMAPF 0  // k_group: the TMA unit bulk-prefetches the next vertex's row into L2
#endif
#ifndef LCC_HDRPF
#define LCC_HDRPF 0  // k_group: vertex headers (list entry, row bounds) loaded ahead
#endif
#ifndef LCC_ROWPF
#define LCC_ROWPF 0  // k_group: prefetch the next vertex's neighbour row into L2 while this one runs
#endif
#ifndef LCC_LK
#define LCC_LK 1  // integer masses: the cluster masses live in the k_group tables (see group_km)
#endif
#ifndef LCC_CLAIMK
#define LCC_CLAIMK 0  // async k_group: the claiming lane gathers the live mass (objective -19% on config 4)
#endif
#ifndef LCC_ASYNC_HINT
#define LCC_ASYNC_HINT 0  // async label / mass loads carry the evict-last L2 policy too
#endif
#ifndef LCC_ILV
#define LCC_ILV 1  // integer-mass rounds: labels and masses interleaved in one (label, mass) array
#endif
#ifndef LCC_KPF
#define LCC_KPF 0  // async k_group: a claim prefetches the cluster's mass into L2 for the scoring-time read
#endif
#ifndef LCC_PACK32
#define LCC_PACK32 1  // async integer-mass rounds with small masses: (label, mass) packed into ONE 32-bit word per vertex
#endif
#ifndef LCC_CODES
#define LCC_CODES 0  // (measured, off) integer-mass async rounds: 4-bit L2-resident codes stand in for the (label, mass) words of own-cluster roots (BMArgs::code)
#endif
#ifndef LCC_MARKBITS
#define LCC_MARKBITS 1  // neighbour marks: 0 byte stores; 1 test-and-set in an n-bit map (L2 resident: config-5 round 116.2 -> 103.6 ms, the byte mask cost ~1.3 G sector write-backs per round); 2 byte stores with the evict-last L2 policy (no effect)
#endif
#ifndef LCC_LK_ASYNC
#define LCC_LK_ASYNC 0  // async rounds too read round-start masses from the packed words (quality -15%)
#endif

constexpr unsigned FULL = 0xffffffffu;
constexpr int SMALL_MAX = 32;
constexpr int SMALL_THREADS = 256;
constexpr int LARGE_CHUNK = 2048;   // edges per insertion work item
constexpr int LARGE_THREADS = 256;
constexpr int SCORE_CHUNK = 16384;  // table slots per scoring work item
constexpr int SCORE_THREADS = 256;

// ---- label / mass gathers ------------------------------------------------
// sync : read-only for the whole kernel -> non-coherent path, L2 evict-last.
// async: other warps store concurrently -> relaxed gpu-scope loads (L2).
template <bool ASYNC>
__device__ __forceinline__ int32_t ldC(const int32_t* C, int64_t i, uint64_t pol) {
    if constexpr (ASYNC) {
        int32_t r;
        if constexpr (LCC_ASYNC_HINT)  // relaxed, with the evict-last L2 policy of the sync path
            asm volatile("ld.relaxed.gpu.global.L2::cache_hint" LCC_PF64 ".s32 %0, [%1], %2;" : "=r"(r) : "l"(C + i), "l"(pol));
        else
            asm volatile("ld.relaxed.gpu.global" LCC_PF64 ".s32 %0, [%1];" : "=r"(r) : "l"(C + i));
        return r;
    } else {
        return ld_keep_i32(C + i, pol);
    }
}
// Integer-mass rounds keep labels and masses interleaved: CK[2v] = C[v],
// CK[2v+1] = mass of cluster v (uint32).  A neighbour's label and -- while
// it is its own cluster, as in every first round -- its cluster's mass then
// share one 8-byte word, so the scoring-time mass gather finds the line the
// label gather already brought into L2 (config 5: the two gathers each
// fetched their own DRAM line, 8x the algorithmic bytes).  a.cs is the
// label stride (2 interleaved, 1 otherwise); KS the mass stride.
constexpr int64_t KS = LCC_ILV ? 2 : 1;
// KI: integer masses, gathered from a uint32 image of K (half the bytes of
// the fp64 array, so labels + masses stay L2-resident); exact, see run_round.
// ks / sh: the image's word stride (2 interleaved, 1 packed or plain) and
// the mass field's shift inside a word (0 unless packed, see BMArgs)
template <bool ASYNC, bool KI>
__device__ __forceinline__ double ldK(const void* Kp, int64_t i, uint64_t pol, int ks = KS, int sh = 0) {
    if constexpr (KI) {
        const uint32_t* K = static_cast<const uint32_t*>(Kp) + ks * i;
        uint32_t r;
        if constexpr (ASYNC && LCC_ASYNC_HINT)
            asm volatile("ld.relaxed.gpu.global.L2::cache_hint" LCC_PF64 ".u32 %0, [%1], %2;" : "=r"(r) : "l"(K), "l"(pol));
        else if constexpr (ASYNC) asm volatile("ld.relaxed.gpu.global" LCC_PF64 ".u32 %0, [%1];" : "=r"(r) : "l"(K));
        else r = (uint32_t)ld_keep_i32(reinterpret_cast<const int32_t*>(K), pol);
        return u32_to_f64(r >> sh);
    } else {
        const double* K = static_cast<const double*>(Kp);
        if constexpr (ASYNC) {
            double r;
            asm volatile("ld.relaxed.gpu.global" LCC_PF64 ".f64 %0, [%1];" : "=d"(r) : "l"(K + i));
            return r;
        } else {
            return ld_keep_f64(K + i, pol);
        }
    }
}
// relaxed mass update; returns the mass before the add
template <bool KI>
__device__ __forceinline__ double addK(void* Kp, int64_t i, double kv, int ks = KS, int sh = 0) {
    if constexpr (KI) return u32_to_f64(atomicAdd(static_cast<uint32_t*>(Kp) + ks * i, (uint32_t)kv << sh) >> sh);
    else return atomicAdd(static_cast<double*>(Kp) + i, kv);
}
template <bool KI>
__device__ __forceinline__ void subK(void* Kp, int64_t i, double kv, int ks = KS, int sh = 0) {
    if constexpr (KI) atomicSub(static_cast<uint32_t*>(Kp) + ks * i, (uint32_t)kv << sh);
    else atomicAdd(static_cast<double*>(Kp) + i, -kv);
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
    void* K;      // double[n | 2n], or the uint32 image (KI kernels)
    int32_t* D;
    uint8_t* moved;
    unsigned long long* moved_count;
    int32_t n;
    uint8_t* mark;  // optional: neighbours of movers flagged here (fused VertexNeighbors frontier)
    const uint8_t* prev_moved;       // async damping (AsyncDamp), or null
    uint32_t salt;
    unsigned long long* pending;     // deferred movers this round
    // packed (label | mass << 32) per vertex, built from C and the uint32
    // mass image at the start of an integer-mass round (KI); null otherwise.
    // Async movers keep their own word current (label and the target's mass
    // after their join); the other members' masses are round-start values.
    unsigned long long* LK;
    int32_t cs;  // label stride in C: 2 when interleaved with the masses (KI rounds), else 1
    // the round's n-byte frontier mask: deferred async movers set their own
    // entry here; `mark` (above) is the same array when movers push their
    // neighbours inside the kernels, null when the marks are pulled after
    // the round (k_pull_head / k_pull_rest)
    uint8_t* dmark;
    // LCC_MARKBITS=1: the neighbour marks go to this n-bit map during the
    // kernels (test, then RED.OR) and are expanded into `mark` after them
    unsigned* mbits;
    // Packed rounds (LCC_PACK32; asynchronous, integer masses, every mass and
    // k_v small): C and K are ONE array of 32-bit words, word i = label of
    // vertex i in the low `ksh` bits | mass of cluster i above them -- half the
    // bytes of the interleaved image, so twice as many vertices per L2 byte.
    // lm masks a loaded label (all ones otherwise); ks is the mass stride in
    // words; ksh the mass shift (0 = not packed); kmax the largest mass a
    // join may produce (a join beyond it is refused like a failed check).
    int32_t lm;
    int32_t ks;
    int32_t ksh;
    double kmax;
    // Codes (LCC_CODES; packed rounds only): 4 bits per vertex, code[i] = the
    // mass of cluster i while word i still reads (label i | mass << ksh) with
    // 1 <= mass <= 15, else 0 -- an L2-resident summary (n/2 bytes) of the
    // packed words: a gather whose code is set needs no DRAM access.  A mover
    // clears the codes of the words it is about to change (its own, its old
    // and its new cluster's) before it changes them, and nothing sets a code
    // during a round, so a set code is never newer than its word: readers see
    // the same relaxed, possibly stale view as with the words alone.
    unsigned* code;
};
// a vertex stores its new label: its word's mass field belongs to the
// cluster of the same id and must survive (packed: add the label difference;
// only v itself ever writes v's label)
__device__ __forceinline__ void stC_own(const BMArgs& a, int32_t v, int32_t c_old, int32_t x);

// packed-word gathers: frozen in sync rounds, relaxed loads in async ones
template <bool ASYNC>
__device__ __forceinline__ unsigned long long ldLK(const unsigned long long* LK, int64_t i, uint64_t pol) {
    unsigned long long r;
    if constexpr (ASYNC) asm volatile("ld.relaxed.gpu.global" LCC_PF64 ".u64 %0, [%1];" : "=l"(r) : "l"(LK + i));
    else asm volatile("ld.global.nc.L2::cache_hint" LCC_PF64 ".u64 %0, [%1], %2;" : "=l"(r) : "l"(LK + i), "l"(pol));
    return r;
}
__device__ __forceinline__ void stLK(unsigned long long* LK, int64_t i, int32_t x, double mass) {
    const unsigned long long w = (unsigned long long)(uint32_t)x | ((unsigned long long)(uint32_t)mass << 32);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(LK + i), "l"(w) : "memory");
}

__device__ __forceinline__ void stC_own(const BMArgs& a, int32_t v, int32_t c_old, int32_t x) {
    if (a.ksh) atomicAdd(reinterpret_cast<uint32_t*>(a.C) + v, (uint32_t)x - (uint32_t)c_old);
    else stC_relaxed(a.C, (int64_t)v * a.cs, x);
}
// ---- codes (see BMArgs::code) ---------------------------------------------
__device__ __forceinline__ uint32_t code_of(const unsigned* code, int32_t i) {
    uint32_t w;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(w) : "l"(code + ((uint32_t)i >> 3)));
    return (w >> (((uint32_t)i & 7u) * 4u)) & 15u;
}
__device__ __forceinline__ void code_clear(const BMArgs& a, int32_t i) {
    if (!LCC_CODES || !a.code || i >= a.n) return;
    unsigned* w = a.code + ((uint32_t)i >> 3);
    const unsigned m = 15u << (((uint32_t)i & 7u) * 4u);
    unsigned cur;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(w));
    if (cur & m) atomicAnd(w, ~m);
}
// label of vertex u / mass of cluster x: from the code when it is set
template <bool ASYNC>
__device__ __forceinline__ int32_t ldLabel(const BMArgs& a, int32_t u, uint64_t pol) {
    if constexpr (ASYNC && LCC_CODES) {
        if (a.code && code_of(a.code, u)) return u;
    }
    return ldC<ASYNC>(a.C, (int64_t)u * a.cs, pol) & a.lm;
}
template <bool ASYNC, bool KI>
__device__ __forceinline__ double ldMass(const BMArgs& a, int32_t x, uint64_t pol) {
    if constexpr (ASYNC && KI && LCC_CODES) {
        if (a.code && x < a.n) {
            const uint32_t cd = code_of(a.code, x);
            if (cd) return u32_to_f64(cd);
        }
    }
    return ldK<ASYNC, KI>(a.K, x, pol, a.ks, a.ksh);
}
// a mover flags neighbour u for the next frontier
__device__ __forceinline__ void mark_nbr(const BMArgs& a, int32_t u) {
#if LCC_MARKBITS == 1
    unsigned* w = a.mbits + ((uint32_t)u >> 5);
    const unsigned bit = 1u << ((uint32_t)u & 31u);
    unsigned cur;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(w));
    if (!(cur & bit)) atomicOr(w, bit);
#elif LCC_MARKBITS == 2
    asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(a.mark + u), "h"((unsigned short)1), "l"(policy_evict_last()) : "memory");
#else
    a.mark[u] = 1;
#endif
}

// Final choice for one vertex (mirrors oracle best_target()).
template <bool ASYNC, bool KI>
__device__ __forceinline__ int decide(const BMArgs& a, int32_t v, int32_t c, double kv, double b,
                                      bool has, double bg, int32_t bx, double bS = NAN) {
    const double gf = dsub(0.0, b);
    int32_t choice = c;
    double cg = 0.0;
    if (has) { choice = bx; cg = bg; }
    if (!has || gf > cg) { choice = a.n + v; cg = gf; }
    if (cg > 0.0) {
        if constexpr (ASYNC) {
            if (a.prev_moved && a.prev_moved[v] && (hash32((uint32_t)v * 0x9E3779B9u + a.salt) & 1u)) {
                // deferred: v moved last iteration too; it stays in the frontier
                a.dmark[v] = 1;
                atomicAdd(a.pending, 1ull);
                return 0;
            }
            if (KI && a.ksh) {
                // packed word: the join is a compare-and-swap on the target's
                // word, so the mass field never holds more than the joins that
                // passed (an add-then-back-out could wrap a 4-5 bit field under
                // contention); a joiner re-reads and re-checks until its swap
                // lands or its gain is gone
                uint32_t* W = static_cast<uint32_t*>(a.K);
                const uint32_t add = (uint32_t)kv << a.ksh;
                if (choice != a.n + v) {
                    code_clear(a, choice);  // before the word changes (BMArgs::code)
                    uint32_t old;
                    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(old) : "l"(W + choice));
                    while (true) {
                        const double kold = u32_to_f64(old >> a.ksh);
                        if (LCC_VALIDATE && bS == bS) {
                            const double gnow = dsub(dsub(bS, dmul(dmul(a.lam, kv), kold)), b);
                            if (!(gnow > 0.0)) return 0;
                        }
                        if (kold + kv > a.kmax) return 0;  // field full: no move this round
                        const uint32_t prev = atomicCAS(W + choice, old, old + add);
                        if (prev == old) break;
                        old = prev;
                    }
                } else {
                    atomicAdd(W + choice, add);  // v's own fresh id: mass 0 -> k_v
                }
                code_clear(a, v);
                code_clear(a, c);
                stC_own(a, v, c, choice);
                atomicSub(W + c, add);
                a.moved[v] = 1;
                return 1;
            }
            if (LCC_VALIDATE && choice != a.n + v && bS == bS) {
                // commit-time check: the mass x has when v joins (the atomic's
                // return value, after every earlier joiner) must still leave a
                // positive gain; otherwise v stays (it is in the next frontier,
                // since its neighbours moved).  Stops stale-mass pile-ups.
                code_clear(a, choice);  // before the word changes (BMArgs::code)
                const double kold = addK<KI>(a.K, choice, kv, a.ks, a.ksh);
                const double gnow = dsub(dsub(bS, dmul(dmul(a.lam, kv), kold)), b);
                if (!(gnow > 0.0)) {
                    subK<KI>(a.K, choice, kv, a.ks, a.ksh);
                    return 0;
                }
                code_clear(a, v);
                code_clear(a, c);
                stC_own(a, v, c, choice);
                if (KI && a.LK) stLK(a.LK, v, choice, kold + kv);
                subK<KI>(a.K, c, kv, a.ks, a.ksh);
                a.moved[v] = 1;
                return 1;
            }
            code_clear(a, choice);
            code_clear(a, v);
            code_clear(a, c);
            stC_own(a, v, c, choice);
            subK<KI>(a.K, c, kv, a.ks, a.ksh);
            const double kold = addK<KI>(a.K, choice, kv, a.ks, a.ksh);
            if (KI && a.LK) stLK(a.LK, v, choice, kold + kv);
        } else {
            a.D[v] = choice;
        }
        a.moved[v] = 1;
        return 1;
    }
    return 0;
}

// Warp argmax under better(): largest gain, ties to the lowest cluster id.
// Three warp reductions (REDUX) on an order-preserving integer image of the
// gain -- its high word, its low word among the lanes that hold the largest
// high word, then the smallest id among the lanes that hold the largest gain --
// instead of five shuffle-and-compare rounds on (gain, id[, S]): ~20
// instructions instead of ~65 per vertex (LCC_REDUX_ARGMAX=0: the shuffles).
#ifndef LCC_REDUX_ARGMAX
#define LCC_REDUX_ARGMAX 1
#endif
__device__ __forceinline__ int warp_argmax_lane(double g, int32_t& x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(dadd(g, 0.0));  // -0 -> +0: equal gains, equal keys
    const unsigned long long k = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    const uint32_t hi = (uint32_t)(k >> 32), lo = (uint32_t)k;
    const uint32_t mhi = __reduce_max_sync(FULL, hi);
    const uint32_t mlo = __reduce_max_sync(FULL, hi == mhi ? lo : 0u);
    const bool top = hi == mhi && lo == mlo;
    const uint32_t mx = __reduce_min_sync(FULL, top ? (uint32_t)x : 0xffffffffu);
    const unsigned who = __ballot_sync(FULL, top && (uint32_t)x == mx);
    x = (int32_t)mx;
    return __ffs(who) - 1;
}
__device__ __forceinline__ void warp_argmax(double& g, int32_t& x) {
#if LCC_REDUX_ARGMAX
    const int src = warp_argmax_lane(g, x);
    g = __shfl_sync(FULL, g, src);
#else
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        double og = __shfl_xor_sync(FULL, g, d);
        int32_t ox = __shfl_xor_sync(FULL, x, d);
        if (better(og, ox, g, x)) { g = og; x = ox; }
    }
#endif
}
// ... carrying the winner's neighbour weight S (commit-time validation)
__device__ __forceinline__ void warp_argmax(double& g, int32_t& x, double& S) {
#if LCC_REDUX_ARGMAX
    const int src = warp_argmax_lane(g, x);
    g = __shfl_sync(FULL, g, src);
    S = __shfl_sync(FULL, S, src);
#else
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        double og = __shfl_xor_sync(FULL, g, d);
        int32_t ox = __shfl_xor_sync(FULL, x, d);
        double oS = __shfl_xor_sync(FULL, S, d);
        if (better(og, ox, g, x)) { g = og; x = ox; S = oS; }
    }
#endif
}

__device__ __forceinline__ void flush_moves(const BMArgs& a, unsigned long long mine) {
#pragma unroll
    for (int d = 16; d; d >>= 1) mine += __shfl_xor_sync(FULL, mine, d);
    if (lane_id() == 0 && mine) atomicAdd(a.moved_count, mine);
}

// ===========================================================================
// small bin: deg <= 32, warp-packed edge windows
// ===========================================================================
#ifndef LCC_SMALL_MINB
#define LCC_SMALL_MINB 4  // 64 registers for the pipelined windows, no spill (+1.4% vs 48 registers unpipelined)
#endif
template <class WT, bool ASYNC, bool KI>
__global__ void __launch_bounds__(SMALL_THREADS, LCC_SMALL_MINB)
k_small(BMArgs a, const int32_t* __restrict__ list, int64_t lo, int64_t hi) {
    constexpr int WPB = SMALL_THREADS / 32;
    __shared__ int32_t s_owner[WPB][32];
    __shared__ double s_sc[LCC_SMALL_PIPE ? 1 : WPB][32];
    __shared__ double s_sc2[LCC_SMALL_PIPE ? 2 : 1][WPB][32];  // per-window S_c, double-buffered
    const int wib = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t nb = (hi - lo + 31) / 32;
    const int64_t gw = ((int64_t)blockIdx.x * SMALL_THREADS + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * SMALL_THREADS) >> 5;
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
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
            c = ldLabel<ASYNC>(a, v, pol_keep);
            kv = kval(a.k, v);
            Kc = ldMass<ASYNC, KI>(a, c, pol_keep);
        }
        const double t = dmul(a.lam, kv);
        int32_t incl = deg;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int32_t y = __shfl_up_sync(FULL, incl, d);
            if (lane >= d) incl += y;
        }
        const int32_t excl = incl - deg;

#if LCC_SMALL_PIPE
        // windows are software pipelined: the next window's geometry and
        // index loads are issued before this window is processed, and its
        // label gathers go out while this window waits for its masses
        struct Geo {
            bool inwin, starter, has_edge;
            int end, rs, p, j, nedges;
            unsigned starts;
            int64_t e;
        };
        auto geometry = [&](int base, int buf, Geo& G) {
            const int32_t base_off = __shfl_sync(FULL, excl, base);
            G.inwin = valid && lane >= base && (incl - base_off) <= SMALL_MAX;
            const unsigned winmask = __ballot_sync(FULL, G.inwin);
            G.end = 32 - __clz(winmask);
            G.nedges = __shfl_sync(FULL, incl, G.end - 1) - base_off;
            G.rs = excl - base_off;
            G.starter = G.inwin && deg > 0;
            G.starts = __reduce_or_sync(FULL, G.starter ? (1u << G.rs) : 0u);
            if (G.starter) s_owner[wib][G.rs] = lane;
            if (G.inwin) s_sc2[buf][wib][lane] = 0.0;
            __syncwarp();
            G.has_edge = lane < G.nedges;
            G.p = 0;
            G.j = 0;
            if (G.has_edge) {
                const unsigned m = G.starts & ((2u << lane) - 1u);
                G.p = 31 - __clz(m);
                G.j = s_owner[wib][G.p];
            }
            __syncwarp();  // s_owner is rewritten by the next window's geometry
            const int64_t sj = __shfl_sync(FULL, s, G.j);
            G.e = sj + (lane - G.p);
        };
        Geo G;
        int buf = 0;
        geometry(0, 0, G);
        int32_t nbr = G.has_edge ? ld_stream_i32(a.indices + G.e, pol_stream) : 0;
        int32_t x = G.has_edge ? ldLabel<ASYNC>(a, nbr, pol_keep) : 0;
        while (true) {
            const bool more = G.end < nvalid;
            Geo Gn;
            int32_t nbr_n = 0;
            if (more) {
                geometry(G.end, buf ^ 1, Gn);
                if (Gn.has_edge) nbr_n = ld_stream_i32(a.indices + Gn.e, pol_stream);
            }
            const int j = G.j, p = G.p, rs = G.rs, nedges = G.nedges;
            const bool has_edge = G.has_edge, inwin = G.inwin, starter = G.starter;
            const unsigned starts = G.starts;
            const int32_t cj = __shfl_sync(FULL, c, j);
            const double tj = __shfl_sync(FULL, t, j);
            const double wv = has_edge ? WLoad<WT>::at(a.w, G.e) : 0.0;
            const uint64_t key = has_edge ? (((uint64_t)(uint32_t)j << 32) | (uint32_t)x)
                                          : ((uint64_t)(64 + lane) << 32);
            const unsigned grp = __match_any_sync(FULL, key);
            double S;
            if constexpr (!WLoad<WT>::weighted) {
                S = u32_to_f64(__popc(grp));
            } else {
                S = 0.0;
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const double wq = __shfl_sync(FULL, wv, q);
                    if ((grp >> q) & 1u) S = dadd(S, wq);
                }
            }
            const bool is_leader = has_edge && lane == (__ffs(grp) - 1);
            const bool cand = is_leader && x != cj;
            // mass gather of this window, then the next window's label gather
            const double Kx = cand ? ldMass<ASYNC, KI>(a, x, pol_keep) : 0.0;
            int32_t x_n = 0;
            if (more && Gn.has_edge) x_n = ldLabel<ASYNC>(a, nbr_n, pol_keep);
            if (is_leader && x == cj) s_sc2[buf][wib][j] = S;
            __syncwarp();
            double bv = 0.0;
            if (inwin) bv = dadd(dsub(s_sc2[buf][wib][lane], dmul(t, Kc)), dmul(t, kv));
            const double bj = __shfl_sync(FULL, bv, j);
            double g = -INFINITY;
            int32_t gx = NO_CAND;
            double gS = 0.0;
            if (cand) {
                gS = S;
                g = dsub(dsub(S, dmul(tj, Kx)), bj);
                gx = x;
            }
            int segend = lane + 1;
            if (has_edge) {
                const unsigned above = starts & ~((2u << lane) - 1u);
                segend = above ? __ffs(above) - 1 : nedges;
            }
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double og = __shfl_down_sync(FULL, g, d);
                const int32_t ox = __shfl_down_sync(FULL, gx, d);
                if (lane + d < segend && better(og, ox, g, gx)) { g = og; gx = ox; }
            }
            const int src = starter ? rs : lane;
            const double hg = __shfl_sync(FULL, g, src);
            const int32_t hx = __shfl_sync(FULL, gx, src);
            double hS = NAN;
            if constexpr (ASYNC && LCC_VALIDATE) {
                const int32_t sx = __shfl_sync(FULL, gx, p);
                const unsigned wm = __ballot_sync(FULL, cand && x == sx);
                const unsigned omask = starter ? ((deg >= 32 ? FULL : ((1u << deg) - 1u)) << rs) : 0u;
                const unsigned wo = wm & omask;
                hS = __shfl_sync(FULL, gS, wo ? __ffs(wo) - 1 : lane);
            }
            const int mv = inwin ? decide<ASYNC, KI>(a, v, c, kv, bv, starter && hx != NO_CAND, hg, hx, hS) : 0;
            my_moves += mv;
            if (a.mark) {  // the window's neighbour ids are still in registers
                const int mvj = __shfl_sync(FULL, mv, j);
                if (has_edge && mvj) mark_nbr(a, nbr);
            }
            __syncwarp();  // s_sc2[buf] is zeroed again two windows on
            if (!more) break;
            G = Gn;
            nbr = nbr_n;
            x = x_n;
            buf ^= 1;
        }
#else
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
            int32_t x = 0, nbr = 0;
            double wv = 0.0;
            if (has_edge) {
                const int64_t e = sj + (lane - p);
                nbr = ld_stream_i32(a.indices + e, pol_stream);
                x = ldLabel<ASYNC>(a, nbr, pol_keep);
                wv = WLoad<WT>::at(a.w, e);
            }
            const uint64_t key = has_edge ? (((uint64_t)(uint32_t)j << 32) | (uint32_t)x)
                                          : ((uint64_t)(64 + lane) << 32);
            const unsigned grp = __match_any_sync(FULL, key);
            double S;
            if constexpr (!WLoad<WT>::weighted) {
                S = u32_to_f64(__popc(grp));
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
            double gS = 0.0;
            if (is_leader && x != cj) {
                gS = S;
                g = dsub(dsub(S, dmul(tj, ldMass<ASYNC, KI>(a, x, pol_keep))), bj);
                gx = x;
            }
#if LCC_SMALL_LADDER2
            // segmented argmax: the segment bound comes from the starts
            // bitmask (no shuffled segment ids); the winner's S is fetched
            // once after the ladder instead of riding every step
            int segend = lane + 1;
            if (has_edge) {
                const unsigned above = starts & ~((2u << lane) - 1u);
                segend = above ? __ffs(above) - 1 : nedges;
            }
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double og = __shfl_down_sync(FULL, g, d);
                const int32_t ox = __shfl_down_sync(FULL, gx, d);
                if (lane + d < segend && better(og, ox, g, gx)) { g = og; gx = ox; }
            }
            const int src = starter ? rs : lane;
            const double hg = __shfl_sync(FULL, g, src);
            const int32_t hx = __shfl_sync(FULL, gx, src);
            double hS = NAN;
            if constexpr (ASYNC && LCC_VALIDATE) {
                const int32_t sx = __shfl_sync(FULL, gx, p);  // my segment's winner (head lane p)
                const unsigned wm = __ballot_sync(FULL, is_leader && x != cj && x == sx);
                // the owner's segment: lanes [rs, rs + deg)
                const unsigned omask = starter ? ((deg >= 32 ? FULL : ((1u << deg) - 1u)) << rs) : 0u;
                const unsigned wo = wm & omask;
                const double sw = __shfl_sync(FULL, gS, wo ? __ffs(wo) - 1 : lane);
                hS = sw;
            }
#else
            const int32_t seg = has_edge ? j : 32 + lane;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const double og = __shfl_down_sync(FULL, g, d);
                const int32_t ox = __shfl_down_sync(FULL, gx, d);
                const int32_t os = __shfl_down_sync(FULL, seg, d);
                double oS = 0.0;
                if constexpr (ASYNC && LCC_VALIDATE) oS = __shfl_down_sync(FULL, gS, d);
                if (lane + d < 32 && os == seg && better(og, ox, g, gx)) { g = og; gx = ox; gS = oS; }
            }
            const int src = starter ? rs : lane;
            const double hg = __shfl_sync(FULL, g, src);
            const int32_t hx = __shfl_sync(FULL, gx, src);
            double hS = NAN;
            if constexpr (ASYNC && LCC_VALIDATE) hS = __shfl_sync(FULL, gS, src);
#endif
            const int mv = inwin ? decide<ASYNC, KI>(a, v, c, kv, bv, starter && hx != NO_CAND, hg, hx, hS) : 0;
            my_moves += mv;
            if (a.mark) {  // the window's neighbour ids are still in registers
                const int mvj = __shfl_sync(FULL, mv, j);
                if (has_edge && mvj) mark_nbr(a, nbr);
            }
            base = end;
            __syncwarp();
        }
#endif
    }
    flush_moves(a, my_moves);
}

// ===========================================================================
// tiny bin: 1 <= deg <= TINY_MAX, one THREAD per vertex.  The labels sit in
// registers; distinct clusters are found by pairwise compares, S sums run in
// CSR order (bit-identical to k_small and the oracle, weighted or not), and
// every first occurrence's mass gather is issued before any gain is formed.
// No shuffles or shared memory: every thread's gathers are independent, so a
// warp keeps 32 vertices' loads in flight instead of one 32-edge window.
// ===========================================================================
#ifndef LCC_TINY_MAX
#define LCC_TINY_MAX 8
#endif
constexpr int TINY_MAX = LCC_TINY_MAX;

#ifndef LCC_TINY_MINB
#define LCC_TINY_MINB 4  // 64 registers, no spill: 32 resident warps (+1%)
#endif
template <class WT, bool ASYNC, bool KI>
__global__ void __launch_bounds__(256, LCC_TINY_MINB)
k_tiny(BMArgs a, const int32_t* __restrict__ list, int64_t lo, int64_t hi) {
    using TW = typename WLoad<WT>::TW;
    // masses held raw (uint32 image or fp64) until the gain: fewer registers
    using KR = typename std::conditional<KI, uint32_t, double>::type;
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    unsigned long long my_moves = 0;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = __ldg(list + i);
        const int64_t s = __ldg(a.indptr + v);
        const int deg = (int)(__ldg(a.indptr + v + 1) - s);
        const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
        const double kv = kval(a.k, v);
        const double Kc = ldMass<ASYNC, KI>(a, c, pol_keep);
        int32_t x[TINY_MAX];
        TW w[TINY_MAX];
#pragma unroll
        for (int j = 0; j < TINY_MAX; ++j) {
            x[j] = j < deg ? ld_stream_i32(a.indices + s + j, pol_stream) : -1;
            w[j] = j < deg ? WLoad<WT>::tw(a.w, s + j) : TW(0);
        }
#pragma unroll
        for (int j = 0; j < TINY_MAX; ++j) x[j] = x[j] >= 0 ? ldLabel<ASYNC>(a, x[j], pol_keep) : EMPTY_KEY;
        // first occurrences of each neighbour cluster (other than c)
        unsigned first = 0;
#pragma unroll
        for (int j = 0; j < TINY_MAX; ++j) {
            bool f = x[j] != EMPTY_KEY && x[j] != c;
#pragma unroll
            for (int q = 0; q < j; ++q) f = f && x[q] != x[j];
            first |= (unsigned)f << j;
        }
        KR Kx[TINY_MAX];
#pragma unroll
        for (int j = 0; j < TINY_MAX; ++j) {
            if constexpr (KI) {
                Kx[j] = 0u;
                if ((first >> j) & 1u) {
                    uint32_t cd = 0u;
                    if constexpr (ASYNC && LCC_CODES) {
                        if (a.code && x[j] < a.n) cd = code_of(a.code, x[j]);
                    }
                    if (cd) {
                        Kx[j] = cd;
                    } else {
                        if constexpr (ASYNC) asm volatile("ld.relaxed.gpu.global" LCC_PF64 ".u32 %0, [%1];" : "=r"(Kx[j]) : "l"(static_cast<const uint32_t*>(a.K) + (int64_t)a.ks * x[j]));
                        else Kx[j] = (uint32_t)ld_keep_i32(static_cast<const int32_t*>(a.K) + (int64_t)a.ks * x[j], pol_keep);
                        Kx[j] >>= a.ksh;
                    }
                }
            } else {
                Kx[j] = ((first >> j) & 1u) ? ldK<ASYNC, false>(a.K, x[j], pol_keep, a.ks, a.ksh) : 0.0;
            }
        }
        double sc = 0.0;
#pragma unroll
        for (int j = 0; j < TINY_MAX; ++j)
            if (x[j] == c) sc = dadd(sc, WLoad<WT>::f64(w[j]));
        const double t = dmul(a.lam, kv);
        const double b = dadd(dsub(sc, dmul(t, Kc)), dmul(t, kv));
        double bg = -INFINITY, bS = 0.0;
        int32_t bx = NO_CAND;
#pragma unroll
        for (int j = 0; j < TINY_MAX; ++j) {
            if (!((first >> j) & 1u)) continue;
            double S = 0.0;
#pragma unroll
            for (int q = j; q < TINY_MAX; ++q)
                if (x[q] == x[j]) S = dadd(S, WLoad<WT>::f64(w[q]));
            double K;
            if constexpr (KI) K = u32_to_f64(Kx[j]);
            else K = Kx[j];
            const double g = dsub(dsub(S, dmul(t, K)), b);
            if (better(g, x[j], bg, bx)) { bg = g; bx = x[j]; bS = S; }
        }
        const int mv = decide<ASYNC, KI>(a, v, c, kv, b, bx != NO_CAND, bg, bx, bS);
        my_moves += mv;
        if (a.mark && mv) {  // neighbour ids re-read (L1/L2-hot)
            for (int j = 0; j < deg; ++j) mark_nbr(a, __ldg(a.indices + s + j));
        }
    }
    flush_moves(a, my_moves);
}

// ===========================================================================
// isolated vertices (deg 0): S = 0 for every cluster, so the only candidate is
// the fresh singleton (gain -b), taken when v sits in a heavier cluster
// ===========================================================================
template <bool ASYNC, bool KI>
__global__ void __launch_bounds__(256)
k_isolated(BMArgs a, const int32_t* __restrict__ list, int64_t lo, int64_t hi) {
    const uint64_t pol_keep = policy_evict_last();
    unsigned long long my_moves = 0;
    for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = __ldg(list + i);
        const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
        const double kv = kval(a.k, v);
        const double t = dmul(a.lam, kv);
        const double b = dadd(dsub(0.0, dmul(t, ldMass<ASYNC, KI>(a, c, pol_keep))), dmul(t, kv));
        my_moves += decide<ASYNC, KI>(a, v, c, kv, b, false, 0.0, 0);
    }
    flush_moves(a, my_moves);
}

// ===========================================================================
// neighbour-cluster tables.  One atomic per edge: unweighted graphs pack
// (cluster id, count) into one 64-bit slot, claimed by a 64-bit CAS that
// already carries count 1, bumped by a 64-bit RED otherwise.  Weighted
// graphs claim a 32-bit key by CAS and add the weight with fp64 RED.
// Scoring scans every slot (plain loads) and resets it, so the table is
// clean for the next vertex without a separate clearing pass.
// ===========================================================================
__device__ __forceinline__ uint32_t slot_of(int32_t x, uint32_t cap) {
#if LCC_FHASH
    // Fibonacci hashing: one multiply (cluster ids are vertex ids, dense)
    return (uint32_t)(((uint64_t)((uint32_t)x * 0x9E3779B1u) * cap) >> 32);
#else
    return (uint32_t)(((uint64_t)hash32((uint32_t)x) * cap) >> 32);
#endif
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr uint64_t EMPTY64 = ~0ull;  // key -1 (never a cluster id); memset(0xff)-able

template <bool FSUM>
struct SmemTable;

template <>
struct SmemTable<false> {
    static constexpr int bytes_per_slot = 8;
    uint32_t keys, cnts;  // int32[cap] keys, then u32[cap] counts (native 32-bit shared atomics)
    __device__ __forceinline__ void init_cap(unsigned char* p, uint32_t CAP) {
        cnts = smem_u32(p);
        keys = cnts + 4 * CAP;
    }
    __device__ __forceinline__ void clear(uint32_t q) const {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(keys + 4 * q), "r"(EMPTY_KEY) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(cnts + 4 * q), "r"(0u) : "memory");
    }
    // returns true when this call claimed the slot (first occurrence of x)
    __device__ __forceinline__ bool insert(uint32_t cap, int32_t x, uint32_t add) const {
        uint32_t slot;
        return insert(cap, x, add, slot);
    }
    // Shared-memory atomics cost ~2 cycles per lane (B300_MICROARCH.md
    // "Atomics": ATOMS spread-addr), 64x a plain LDS, and bound the group
    // bins.  So one atomic per edge: the slot's key is read first; a repeat
    // key costs one RED, a fresh key one CAS.  The claimer's own weight is
    // implicit: counts hold (sum of weights - 1) mod 2^32, S = count + 1, so
    // a unit-weight claim needs no RED at all.
    __device__ __forceinline__ bool insert(uint32_t cap, int32_t x, uint32_t add, uint32_t& slot) const {
        uint32_t h = slot_of(x, cap);
#if LCC_LDS_FIRST
        while (true) {
            int32_t kq;
            asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(kq) : "r"(keys + 4 * h));
            if (kq == x) break;
            if (kq == EMPTY_KEY) {
                int32_t prev;
                asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(prev) : "r"(keys + 4 * h), "r"(EMPTY_KEY), "r"(x) : "memory");
                if (prev == EMPTY_KEY) {
                    if (add != 1u) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnts + 4 * h), "r"(add - 1u) : "memory");
                    slot = h;
                    return true;
                }
                if (prev == x) break;
            }
            h = (h + 1 == cap) ? 0 : h + 1;
        }
        asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnts + 4 * h), "r"(add) : "memory");
        slot = h;
        return false;
#else
        int32_t prev;
        while (true) {
            asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(prev) : "r"(keys + 4 * h), "r"(EMPTY_KEY), "r"(x) : "memory");
            if (prev == EMPTY_KEY || prev == x) break;
            h = (h + 1 == cap) ? 0 : h + 1;
        }
        const uint32_t inc = prev == EMPTY_KEY ? add - 1u : add;
        if (inc || LCC_ALWAYS_RED) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnts + 4 * h), "r"(inc) : "memory");
        slot = h;
        return prev == EMPTY_KEY;
#endif
    }
    __device__ __forceinline__ bool take(uint32_t q, int32_t& x, double& S) const {
        int32_t kq;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(kq) : "r"(keys + 4 * q));
        if (kq == EMPTY_KEY) return false;
        uint32_t cq;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cq) : "r"(cnts + 4 * q));
        clear(q);
        x = kq;
        S = u32_to_f64(cq + 1u);
        return true;
    }
};

template <>
struct SmemTable<true> {
    static constexpr int bytes_per_slot = 12;
    uint32_t keys, vals;  // int32[cap] keys, then double[cap] sums (8B aligned)
    uint32_t capmax;
    __device__ __forceinline__ void init_cap(unsigned char* p, uint32_t CAP) {
        vals = smem_u32(p);
        keys = vals + 8 * CAP;
        capmax = CAP;
    }
    __device__ __forceinline__ void clear(uint32_t q) const {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(keys + 4 * q), "r"(EMPTY_KEY) : "memory");
        asm volatile("st.shared.f64 [%0], %1;" ::"r"(vals + 8 * q), "d"(0.0) : "memory");
    }
    __device__ __forceinline__ bool insert(uint32_t cap, int32_t x, double wv) const {
        uint32_t slot;
        return insert(cap, x, wv, slot);
    }
    __device__ __forceinline__ bool insert(uint32_t cap, int32_t x, double wv, uint32_t& slot) const {
        uint32_t h = slot_of(x, cap);
        bool fresh = false;
        while (true) {
            int32_t kq;
            asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(kq) : "r"(keys + 4 * h));
            if (kq == x) break;
            if (kq == EMPTY_KEY) {
                int32_t prev;
                asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(prev) : "r"(keys + 4 * h), "r"(EMPTY_KEY), "r"(x) : "memory");
                fresh = prev == EMPTY_KEY;
                if (prev == EMPTY_KEY || prev == x) break;
            }
            h = (h + 1 == cap) ? 0 : h + 1;
        }
        asm volatile("red.shared.add.f64 [%0], %1;" ::"r"(vals + 8 * h), "d"(wv) : "memory");
        slot = h;
        return fresh;
    }
        __device__ __forceinline__ bool take(uint32_t q, int32_t& x, double& S) const {
        int32_t kq;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(kq) : "r"(keys + 4 * q));
        if (kq == EMPTY_KEY) return false;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(S) : "r"(vals + 8 * q));
        clear(q);
        x = kq;
        return true;
    }
};

// integer counts plus the cluster's mass, stored by the claiming lane (it
// arrives with the label in the packed LK word): scoring reads no global
// memory.  12 bytes per slot.
struct SmemTableKM {
    static constexpr int bytes_per_slot = 12;
    uint32_t keys, cnts, mass;
    __device__ __forceinline__ void init_cap(unsigned char* p, uint32_t CAP) {
        cnts = smem_u32(p);
        keys = cnts + 4 * CAP;
        mass = keys + 4 * CAP;
    }
    __device__ __forceinline__ void clear(uint32_t q) const {
        asm volatile("st.shared.b32 [%0], %1;" ::"r"(keys + 4 * q), "r"(EMPTY_KEY) : "memory");
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(cnts + 4 * q), "r"(0u) : "memory");
    }
    __device__ __forceinline__ void insert(uint32_t cap, int32_t x, uint32_t add, uint32_t m) const {
        uint32_t h = slot_of(x, cap);
        int32_t prev;
        while (true) {
            asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(prev) : "r"(keys + 4 * h), "r"(EMPTY_KEY), "r"(x) : "memory");
            if (prev == EMPTY_KEY || prev == x) break;
            h = (h + 1 == cap) ? 0 : h + 1;
        }
        if (prev == EMPTY_KEY) {
            asm volatile("st.shared.u32 [%0], %1;" ::"r"(mass + 4 * h), "r"(m) : "memory");
            if (add != 1u) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnts + 4 * h), "r"(add - 1u) : "memory");
        } else {
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnts + 4 * h), "r"(add) : "memory");
        }
    }
    // claim-or-add without the mass: returns true (and the slot) for a claim
    __device__ __forceinline__ bool insert_claim(uint32_t cap, int32_t x, uint32_t add, uint32_t& slot) const {
        uint32_t h = slot_of(x, cap);
        int32_t prev;
        while (true) {
            asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(prev) : "r"(keys + 4 * h), "r"(EMPTY_KEY), "r"(x) : "memory");
            if (prev == EMPTY_KEY || prev == x) break;
            h = (h + 1 == cap) ? 0 : h + 1;
        }
        const uint32_t inc = prev == EMPTY_KEY ? add - 1u : add;
        if (inc) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnts + 4 * h), "r"(inc) : "memory");
        slot = h;
        return prev == EMPTY_KEY;
    }
    __device__ __forceinline__ void set_mass(uint32_t q, uint32_t m) const {
        asm volatile("st.shared.u32 [%0], %1;" ::"r"(mass + 4 * q), "r"(m) : "memory");
    }
    __device__ __forceinline__ bool take(uint32_t q, int32_t& x, double& S, double& K) const {
        int32_t kq;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(kq) : "r"(keys + 4 * q));
        if (kq == EMPTY_KEY) return false;
        uint32_t cq, mq;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cq) : "r"(cnts + 4 * q));
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(mq) : "r"(mass + 4 * q));
        clear(q);
        x = kq;
        S = u32_to_f64(cq + 1u);
        K = u32_to_f64(mq);
        return true;
    }
};

// global-memory (L2-resident) variant for hubs: same packing, device atomics
template <bool WEIGHTED>
struct GlobalTable;
template <>
struct GlobalTable<false> {
    static constexpr int bytes_per_slot = 8;
    unsigned long long* tab;
    __device__ __forceinline__ void insert(uint32_t cap, int32_t x, uint32_t add) const {
        uint32_t h = slot_of(x, cap);
        const unsigned long long want = ((unsigned long long)(uint32_t)x << 32) | add;
        while (true) {
            const unsigned long long prev = atomicCAS(tab + h, (unsigned long long)EMPTY64, want);
            if (prev == EMPTY64) return;
            if ((int32_t)(prev >> 32) == x) {
                atomicAdd(tab + h, (unsigned long long)add);
                return;
            }
            h = (h + 1 == cap) ? 0 : h + 1;
        }
    }
    __device__ __forceinline__ bool read(uint32_t q, int32_t& x, double& S) const {
        const unsigned long long w = tab[q];
        if (w == EMPTY64) return false;
        x = (int32_t)(w >> 32);
        S = u32_to_f64((uint32_t)w);
        return true;
    }
    __device__ __forceinline__ double find(uint32_t cap, int32_t x) const {
        for (uint32_t h = slot_of(x, cap);; h = (h + 1 == cap) ? 0 : h + 1) {
            const unsigned long long w = tab[h];
            if (w == EMPTY64) return NAN;
            if ((int32_t)(w >> 32) == x) return u32_to_f64((uint32_t)w);
        }
    }
};
template <>
struct GlobalTable<true> {
    static constexpr int bytes_per_slot = 12;
    int32_t* keys;
    double* vals;
    __device__ __forceinline__ void insert(uint32_t cap, int32_t x, double wv) const {
        uint32_t h = slot_of(x, cap);
        while (true) {
            const int32_t prev = atomicCAS(keys + h, EMPTY_KEY, x);
            if (prev == EMPTY_KEY || prev == x) break;
            h = (h + 1 == cap) ? 0 : h + 1;
        }
        atomicAdd(vals + h, wv);
    }
    __device__ __forceinline__ bool read(uint32_t q, int32_t& x, double& S) const {
        const int32_t kq = keys[q];
        if (kq == EMPTY_KEY) return false;
        x = kq;
        S = vals[q];
        return true;
    }
    __device__ __forceinline__ double find(uint32_t cap, int32_t x) const {
        for (uint32_t h = slot_of(x, cap);; h = (h + 1 == cap) ? 0 : h + 1) {
            const int32_t kq = keys[h];
            if (kq == EMPTY_KEY) return NAN;
            if (kq == x) return vals[h];
        }
    }
};

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ===========================================================================
// group bins: GW warps per vertex, CAP-slot shared-memory table per group.
// Every lane keeps U independent loads in flight (index stream + label
// gather; then slot read + mass gather) before consuming them.
// ===========================================================================
// Integer masses (KI) and integer sums: the cluster's mass goes into the
// table with the claim, so scoring reads no global memory.
//   sync : the mass comes with the label in one packed gather (LK: frozen
//          labels and masses, exact);
//   async: masses must be read late: a live gather at claim time measured
//          271K instead of 333K objective on config 4 (round-start masses
//          285K), so async rounds keep the scoring-time mass gather
//          (LCC_CLAIMK=1 selects the claim-time variant for experiments).
template <class WT, bool ASYNC, bool KI>
constexpr bool group_km() { return KI && !WLoad<WT>::fsum && LCC_LK && (!ASYNC || LCC_LK_ASYNC || LCC_CLAIMK); }
template <class WT, bool ASYNC, bool KI>
constexpr bool group_lk() { return group_km<WT, ASYNC, KI>() && (!ASYNC || LCC_LK_ASYNC); }
template <class WT, bool ASYNC, bool KI>
using GroupTable = std::conditional_t<group_km<WT, ASYNC, KI>(), SmemTableKM, SmemTable<WLoad<WT>::fsum>>;
template <class WT, bool ASYNC, bool KI, int CAP, int GROUPS>
constexpr size_t group_smem_bytes() {
    return (size_t)GROUPS * CAP * GroupTable<WT, ASYNC, KI>::bytes_per_slot;
}

template <class WT, bool ASYNC, bool KI, int GW, int CAP, int GROUPS, int U, int MINB = 1>
__global__ void __launch_bounds__(GW * 32 * GROUPS, MINB)
k_group(BMArgs a, const int32_t* __restrict__ list, int64_t lo, int64_t hi) {
    constexpr bool FSUM = WLoad<WT>::fsum;
    constexpr bool KM = group_km<WT, ASYNC, KI>();    // masses in the table
    constexpr bool LKP = group_lk<WT, ASYNC, KI>();   // ... from packed (label, mass) gathers
    constexpr bool CLAIMK = KM && !LKP;               // ... gathered live by the claiming lane
    using TW = typename WLoad<WT>::TW;
    using Tab = GroupTable<WT, ASYNC, KI>;
    constexpr int GT = GW * 32;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_g[GROUPS * GW];
    __shared__ double s_scp[GW > 1 ? GROUPS * GW : 1];  // S_c partials (own array: no reuse barrier)
    __shared__ int32_t s_x[GROUPS * GW];
    __shared__ int32_t s_mv[GROUPS];
    constexpr bool VAL = ASYNC && LCC_VALIDATE;
    __shared__ double s_S[VAL ? GROUPS * GW : 1];
    const int gid = threadIdx.x / GT;
    const int gt = threadIdx.x % GT;
    const int wig = gt >> 5;
    const int lane = threadIdx.x & 31;
    Tab tab;
    tab.init_cap(smem + (size_t)gid * CAP * Tab::bytes_per_slot, CAP);
    auto gsync = [&]() {
        if constexpr (GW == 1) __syncwarp();
        else named_sync(1 + gid, GT);
    };
    for (uint32_t q = gt; q < CAP; q += GT) tab.clear(q);
    gsync();
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    unsigned long long my_moves = 0;
    // multi-warp groups: two barriers per vertex (after the inserts, after the
    // argmax partials); the previous vertex's movers flag their neighbours
    // right after the next vertex's first barrier (s_mv is stable there)
    int64_t prev_s = 0, prev_e = 0;
    bool prev_pending = false;
    auto mark_prev = [&]() {
        if (a.mark && prev_pending && s_mv[gid]) {
#pragma unroll 4
            for (int64_t e = prev_s + gt; e < prev_e; e += GT) mark_nbr(a, __ldg(a.indices + e));
        }
    };
    // vertex headers one vertex ahead (LCC_HDRPF): the next vertex's list
    // entry two steps ahead, its row bounds one step ahead, so a vertex's
    // first index loads do not wait on the list -> indptr chain
    const int64_t vstep = (int64_t)gridDim.x * GROUPS;
    int32_t v_nx = 0, v_nn = 0;
    int64_t s_nx = 0, e_nx = 0;
    if constexpr (LCC_HDRPF) {
        const int64_t i0 = lo + (int64_t)blockIdx.x * GROUPS + gid;
        if (i0 < hi) {
            v_nx = __ldg(list + i0);
            s_nx = __ldg(a.indptr + v_nx);
            e_nx = __ldg(a.indptr + v_nx + 1);
        }
        if (i0 + vstep < hi) v_nn = __ldg(list + i0 + vstep);
    }
    for (int64_t i = lo + (int64_t)blockIdx.x * GROUPS + gid; i < hi; i += vstep) {
        int32_t v;
        int64_t s, end;
        if constexpr (LCC_HDRPF) {
            v = v_nx;
            s = s_nx;
            end = e_nx;
            if (i + vstep < hi) {
                v_nx = v_nn;
                s_nx = __ldg(a.indptr + v_nx);
                e_nx = __ldg(a.indptr + v_nx + 1);
                if (i + 2 * vstep < hi) v_nn = __ldg(list + i + 2 * vstep);
            }
        } else {
            v = __ldg(list + i);
            s = __ldg(a.indptr + v);
            end = __ldg(a.indptr + v + 1);
        }
        const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
        const int64_t deg = end - s;
        const uint32_t cap = (uint32_t)min64(CAP, (2 * deg + 31) & ~31LL);
        if constexpr (LCC_TMAPF) {
            // one cp.async.bulk.prefetch.L2 per row, issued by the group's
            // first lane: the next vertex's index row is on its way to L2
            // while this vertex runs (16-byte aligned, size a multiple of 16)
            const int64_t in = i + (int64_t)gridDim.x * GROUPS;
            if (gt == 0 && in < hi) {
                const int32_t vn = __ldg(list + in);
                const int64_t sn = __ldg(a.indptr + vn), en = __ldg(a.indptr + vn + 1);
                const uintptr_t b0 = (uintptr_t)(a.indices + sn) & ~(uintptr_t)15;
                const uintptr_t b1 = ((uintptr_t)(a.indices + en) + 15) & ~(uintptr_t)15;
                if (b1 > b0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(b0), "r"((uint32_t)(b1 - b0)) : "memory");
            }
        }
        if constexpr (LCC_ROWPF) {
            // the group's next vertex: its index row is streamed into L2 now,
            // so that vertex's index loads leave the dependent chain
            const int64_t in = i + (int64_t)gridDim.x * GROUPS;
            if (in < hi) {
                const int32_t vn = __ldg(list + in);
                const int64_t sn = __ldg(a.indptr + vn), en = __ldg(a.indptr + vn + 1);
                const char* base = reinterpret_cast<const char*>(a.indices + sn);
                const int64_t lines = ((en - sn) * 4 + ((uintptr_t)base & 127) + 127) >> 7;
                const char* b0 = reinterpret_cast<const char*>((uintptr_t)base & ~(uintptr_t)127);
                for (int64_t l = gt; l < lines; l += GT) asm volatile("prefetch.global.L2::evict_normal [%0];" ::"l"(b0 + (l << 7)));
            }
        }
        const double kv = kval(a.k, v);
        const double Kc = ldMass<ASYNC, KI>(a, c, pol_keep);
        const double t = dmul(a.lam, kv);
        double sc = 0.0;  // S_c: weight to v's own cluster (kept out of the table)
        for (int64_t e0 = s + gt; e0 < end; e0 += (int64_t)GT * U) {
            int32_t u[U];
            TW wv[U];
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const int64_t e = e0 + (int64_t)j * GT;
                u[j] = e < end ? ld_stream_i32(a.indices + e, pol_stream) : -1;
                wv[j] = e < end ? WLoad<WT>::tw(a.w, e) : TW(0);
            }
            if constexpr (LKP) {
                // one gather per edge: the neighbour's packed (label, mass)
                unsigned long long lk[U];
#pragma unroll
                for (int j = 0; j < U; ++j) lk[j] = u[j] >= 0 ? ldLK<ASYNC>(a.LK, u[j], pol_keep) : ~0ull;
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    if (lk[j] == ~0ull) continue;
                    const int32_t x = (int32_t)(uint32_t)lk[j];
                    if (x == c) sc += WLoad<WT>::f64(wv[j]);
                    else tab.insert(cap, x, (uint32_t)wv[j], (uint32_t)(lk[j] >> 32));
                }
            } else if constexpr (CLAIMK) {
#pragma unroll
                for (int j = 0; j < U; ++j) u[j] = u[j] >= 0 ? ldLabel<ASYNC>(a, u[j], pol_keep) : EMPTY_KEY;
                uint32_t slot[U];
                bool cl[U];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    cl[j] = false;
                    if (u[j] == EMPTY_KEY) continue;
                    if (u[j] == c) sc += WLoad<WT>::f64(wv[j]);
                    else cl[j] = tab.insert_claim(cap, u[j], (uint32_t)wv[j], slot[j]);
                }
                // the claims' live masses: issued together, stored after
                uint32_t km[U];
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    if (cl[j]) asm volatile("ld.relaxed.gpu.global" LCC_PF64 ".u32 %0, [%1];" : "=r"(km[j])
                                            : "l"(static_cast<const uint32_t*>(a.K) + KS * u[j]));
                }
#pragma unroll
                for (int j = 0; j < U; ++j)
                    if (cl[j]) tab.set_mass(slot[j], km[j]);
            } else {
#pragma unroll
            for (int j = 0; j < U; ++j) u[j] = u[j] >= 0 ? ldLabel<ASYNC>(a, u[j], pol_keep) : EMPTY_KEY;
            // (batched probe rounds measured slower here than for the L2
            // tables: shared-memory CAS latency is short, registers are not)
#pragma unroll
            for (int j = 0; j < U; ++j) {
                if (u[j] == EMPTY_KEY) continue;
                if (u[j] == c) {
                    sc += WLoad<WT>::f64(wv[j]);
                } else {
                    const bool claimed = tab.insert(cap, u[j], wv[j]);
                    if constexpr (LCC_KPF && KI) {
                        // the scoring pass reads this mass live; start its trip to L2 now
                        if (claimed) asm volatile("prefetch.global.L2 [%0];" ::"l"(static_cast<const uint32_t*>(a.K) + KS * u[j]));
                    }
                }
            }
            }
        }
        if constexpr (!FSUM && LCC_REDUX_ARGMAX) {
            // integer sums (< 2^32, see best_moves_round): one REDUX instead of five shuffle-adds
            sc = u32_to_f64(__reduce_add_sync(FULL, (uint32_t)sc));
        } else {
#pragma unroll
            for (int d = 16; d; d >>= 1) sc += __shfl_xor_sync(FULL, sc, d);
        }
        if constexpr (GW > 1) {
            if (lane == 0) s_scp[gid * GW + wig] = sc;
        }
        gsync();  // (A) table complete, S_c partials and the previous vertex's s_mv visible
        if constexpr (GW > 1) {
            mark_prev();
            sc = 0.0;
#pragma unroll
            for (int w = 0; w < GW; ++w) sc += s_scp[gid * GW + w];
        }
        const double b = dadd(dsub(sc, dmul(t, Kc)), dmul(t, kv));
        double bg = -INFINITY;
        int32_t bx = NO_CAND;
        double bS = 0.0;
        for (uint32_t q0 = gt; q0 < cap; q0 += GT * U) {
            int32_t x[U];
            double S[U], Kx[U];
            if constexpr (KM) {
#pragma unroll
                for (int j = 0; j < U; ++j) {
                    const uint32_t q = q0 + j * GT;
                    if (!(q < cap && tab.take(q, x[j], S[j], Kx[j]))) x[j] = EMPTY_KEY;
                }
            } else {
#pragma unroll
            for (int j = 0; j < U; ++j) {
                const uint32_t q = q0 + j * GT;
                if (!(q < cap && tab.take(q, x[j], S[j]))) x[j] = EMPTY_KEY;
            }
#pragma unroll
            for (int j = 0; j < U; ++j) Kx[j] = x[j] != EMPTY_KEY ? ldMass<ASYNC, KI>(a, x[j], pol_keep) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < U; ++j) {
                if (x[j] == EMPTY_KEY) continue;
                const double gq = dsub(dsub(S[j], dmul(t, Kx[j])), b);
                if (better(gq, x[j], bg, bx)) { bg = gq; bx = x[j]; bS = S[j]; }
            }
        }
        if constexpr (VAL) warp_argmax(bg, bx, bS);
        else warp_argmax(bg, bx);
        if constexpr (GW > 1) {
            if (lane == 0) {
                s_g[gid * GW + wig] = bg;
                s_x[gid * GW + wig] = bx;
                if constexpr (VAL) s_S[gid * GW + wig] = bS;
            }
            gsync();  // (B) partials visible; every warp has finished scoring (table clean)
#pragma unroll
            for (int w = 0; w < GW; ++w) {
                const double og = s_g[gid * GW + w];
                const int32_t ox = s_x[gid * GW + w];
                if (better(og, ox, bg, bx)) {
                    bg = og;
                    bx = ox;
                    if constexpr (VAL) bS = s_S[gid * GW + w];
                }
            }
        }
        int mv = 0;
        if (gt == 0) {
            mv = decide<ASYNC, KI>(a, v, c, kv, b, bx != NO_CAND, bg, bx, VAL ? bS : NAN);
            my_moves += mv;
        }
        if constexpr (GW == 1) {
            if (a.mark) {  // fused frontier: a mover flags its neighbours (row re-read hits L2)
                mv = __shfl_sync(FULL, mv, 0);
                if (mv) {
#pragma unroll 4
                    for (int64_t e = s + gt; e < end; e += GT) mark_nbr(a, __ldg(a.indices + e));
                }
            }
            __syncwarp();
        } else {
            // s_mv is read by the group after the next vertex's barrier (A);
            // every reader of this slot passed (B) of this vertex already
            if (gt == 0) s_mv[gid] = mv;
            prev_s = s;
            prev_e = end;
            prev_pending = true;
        }
    }
    if constexpr (GW > 1) {
        gsync();
        mark_prev();
    }
    flush_moves(a, my_moves);
}

// ===========================================================================
// window bin (33 <= deg < T <= 512): edge-balanced multi-vertex CTAs.
// The bin list is cut into windows along its degree prefix (window w = list
// entries whose prefix falls in [w*W, (w+1)*W)), so every CTA does the same
// edge work whatever the degree mix and no vertex straddles two CTAs
// (deg < W).  A window holds <= 2W-1 edges and <= 31 vertices, so a table key
// packs (vertex slot, cluster id) into 32 bits and every shared-memory atomic
// is a native 32-bit one (64-bit shared CAS is emulated by a spin loop).
//   1. each thread takes 8 consecutive edge positions: index loads, label
//      gathers (8 in flight), then insert key -> count (CAS + RED per edge);
//      edges into the vertex's own cluster add to S_c instead;
//   2. every slot is scored; per-vertex argmax in three 32-bit atomic steps
//      (max of the high word of the order-preserving gain bits, max of the low
//      word among those, min cluster id among exact maxima: lowest-id ties);
//   3. one thread per vertex decides.
// ===========================================================================
constexpr int WIN_THREADS = 128;
constexpr int WIN_ITEMS = 8;
constexpr int WIN_W = WIN_THREADS * WIN_ITEMS / 2;  // 512: window edges <= 2W-1 = 1023
constexpr int WIN_CAP = 2048;                       // table slots: load <= 0.5
constexpr int WIN_MAXV = 32;                        // (2W-1)/33 + 1 = 31 vertices max
constexpr int LABEL_BITS = 27;                      // cluster ids < 2^27 (n < 2^26)
constexpr uint32_t KEY_EMPTY = 0xffffffffu;

__device__ __forceinline__ unsigned long long ord_gain(double g) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(g);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double unord_gain(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)b);
}

template <bool FSUM>
constexpr size_t window_smem_bytes() {
    // keys u32 + counts u32 (or sums f64) + gain f64
    return (size_t)WIN_CAP * (4 + (FSUM ? 8 : 4) + 8);
}

template <class WT, bool ASYNC, bool KI>
__global__ void __launch_bounds__(WIN_THREADS)
k_window(BMArgs a, const int32_t* __restrict__ list, const int64_t* __restrict__ off,
         const int64_t* __restrict__ wstart, int64_t w0, int64_t w1) {
    constexpr bool FSUM = WLoad<WT>::fsum;
    using TW = typename WLoad<WT>::TW;
    extern __shared__ __align__(16) unsigned char smem[];
    double* gval = reinterpret_cast<double*>(smem);
    double* sums = reinterpret_cast<double*>(smem + (size_t)WIN_CAP * 8);          // weighted
    uint32_t* cnts = reinterpret_cast<uint32_t*>(smem + (size_t)WIN_CAP * 8);      // unweighted
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem + (size_t)WIN_CAP * (FSUM ? 16 : 12));
    __shared__ int64_t s_start[WIN_MAXV];
    __shared__ int32_t s_loc[WIN_MAXV + 1];
    __shared__ int32_t s_v[WIN_MAXV], s_c[WIN_MAXV];
    __shared__ double s_t[WIN_MAXV], s_kv[WIN_MAXV], s_Kc[WIN_MAXV], s_b[WIN_MAXV], s_scw[WIN_MAXV];
    __shared__ uint32_t s_sc[WIN_MAXV], s_hi[WIN_MAXV], s_lo[WIN_MAXV];
    __shared__ int32_t s_bx[WIN_MAXV];
    __shared__ int32_t s_mv[WIN_MAXV];
    const int tid = threadIdx.x;
    const uint32_t keys_s = smem_u32(keys), cnts_s = smem_u32(cnts), sums_s = smem_u32(sums);
    for (int q = tid; q < WIN_CAP; q += WIN_THREADS) {
        keys[q] = KEY_EMPTY;
        if constexpr (FSUM) sums[q] = 0.0;
        else cnts[q] = 0;
    }
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    unsigned long long my_moves = 0;
    for (int64_t w = w0 + blockIdx.x; w < w1; w += gridDim.x) {
        const int64_t i0 = __ldg(wstart + w), i1 = __ldg(wstart + w + 1);
        const int nv = (int)(i1 - i0);
        if (nv <= 0) continue;  // uniform across the CTA
        const int64_t base = __ldg(off + i0);
        const int E = (int)(__ldg(off + i1) - base);
        // ---- 0. per-vertex setup
        if (tid < nv) {
            const int32_t v = __ldg(list + i0 + tid);
            s_v[tid] = v;
            s_start[tid] = __ldg(a.indptr + v);
            s_loc[tid] = (int32_t)(__ldg(off + i0 + tid) - base);
            const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
            s_c[tid] = c;
            const double kv = kval(a.k, v);
            s_kv[tid] = kv;
            s_t[tid] = dmul(a.lam, kv);
            s_Kc[tid] = ldMass<ASYNC, KI>(a, c, pol_keep);
            s_sc[tid] = 0;
            s_scw[tid] = 0.0;
            s_hi[tid] = 0;
            s_lo[tid] = 0;
            s_bx[tid] = NO_CAND;
        }
        if (tid == 0) s_loc[nv] = E;
        __syncthreads();
        const uint32_t cap = (uint32_t)min64(WIN_CAP, ((int64_t)2 * E + 127) & ~127LL);
        // ---- 1. edges: 8 consecutive positions per thread
        {
            const int p0 = tid * WIN_ITEMS;
            int32_t u[WIN_ITEMS];
            int slot[WIN_ITEMS];
            TW wv[WIN_ITEMS];
            int sl = 0;
            if (p0 < E) {
                int lo = 0, hi = nv;  // last sl with s_loc[sl] <= p0
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_loc[mid] <= p0) lo = mid; else hi = mid;
                }
                sl = lo;
            }
#pragma unroll
            for (int j = 0; j < WIN_ITEMS; ++j) {
                const int p = p0 + j;
                u[j] = -1;
                wv[j] = TW(0);
                slot[j] = 0;
                if (p < E) {
                    while (p >= s_loc[sl + 1]) ++sl;
                    const int64_t e = s_start[sl] + (p - s_loc[sl]);
                    u[j] = ld_stream_i32(a.indices + e, pol_stream);
                    wv[j] = WLoad<WT>::tw(a.w, e);
                    slot[j] = sl;
                }
            }
#pragma unroll
            for (int j = 0; j < WIN_ITEMS; ++j) u[j] = u[j] >= 0 ? ldLabel<ASYNC>(a, u[j], pol_keep) : EMPTY_KEY;
#pragma unroll
            for (int j = 0; j < WIN_ITEMS; ++j) {
                if (u[j] == EMPTY_KEY) continue;
                const int sj = slot[j];
                if (u[j] == s_c[sj]) {
                    if constexpr (FSUM) atomicAdd(&s_scw[sj], wv[j]);
                    else atomicAdd(&s_sc[sj], wv[j]);
                    continue;
                }
                const uint32_t key = ((uint32_t)sj << LABEL_BITS) | (uint32_t)u[j];
                uint32_t h = (uint32_t)(((uint64_t)hash32(key) * cap) >> 32);
                while (true) {
                    uint32_t prev;
                    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(prev) : "r"(keys_s + 4 * h), "r"(KEY_EMPTY), "r"(key) : "memory");
                    if (prev == KEY_EMPTY || prev == key) break;
                    h = (h + 1 == cap) ? 0 : h + 1;
                }
                if constexpr (FSUM) asm volatile("red.shared.add.f64 [%0], %1;" ::"r"(sums_s + 8 * h), "d"(wv[j]) : "memory");
                else asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(cnts_s + 4 * h), "r"(wv[j]) : "memory");
            }
        }
        __syncthreads();
        if (tid < nv) {
            const double sc = FSUM ? s_scw[tid] : u32_to_f64(s_sc[tid]);
            s_b[tid] = dadd(dsub(sc, dmul(s_t[tid], s_Kc[tid])), dmul(s_t[tid], s_kv[tid]));
        }
        __syncthreads();
        // ---- 2. score every slot; per-vertex max of the high gain word
        for (uint32_t q = tid; q < cap; q += WIN_THREADS) {
            const uint32_t key = keys[q];
            if (key == KEY_EMPTY) continue;
            const int32_t x = (int32_t)(key & ((1u << LABEL_BITS) - 1u));
            const int sj = (int)(key >> LABEL_BITS);
            const double S = FSUM ? sums[q] : u32_to_f64(cnts[q]);
            const double g = dsub(dsub(S, dmul(s_t[sj], ldMass<ASYNC, KI>(a, x, pol_keep))), s_b[sj]);
            gval[q] = g;
            atomicMax(&s_hi[sj], (uint32_t)(ord_gain(g) >> 32));
        }
        __syncthreads();
        for (uint32_t q = tid; q < cap; q += WIN_THREADS) {
            const uint32_t key = keys[q];
            if (key == KEY_EMPTY) continue;
            const int sj = (int)(key >> LABEL_BITS);
            const unsigned long long o = ord_gain(gval[q]);
            if ((uint32_t)(o >> 32) == s_hi[sj]) atomicMax(&s_lo[sj], (uint32_t)o);
        }
        __syncthreads();
        for (uint32_t q = tid; q < cap; q += WIN_THREADS) {
            const uint32_t key = keys[q];
            if (key == KEY_EMPTY) continue;
            const int sj = (int)(key >> LABEL_BITS);
            const unsigned long long o = ord_gain(gval[q]);
            if ((uint32_t)(o >> 32) == s_hi[sj] && (uint32_t)o == s_lo[sj])
                atomicMin(&s_bx[sj], (int32_t)(key & ((1u << LABEL_BITS) - 1u)));
            keys[q] = KEY_EMPTY;  // reset for the next window
            if constexpr (FSUM) sums[q] = 0.0;
            else cnts[q] = 0;
        }
        __syncthreads();
        // ---- 3. decide
        if (tid < nv) {
            const int32_t bx = s_bx[tid];
            const unsigned long long o = ((unsigned long long)s_hi[tid] << 32) | s_lo[tid];
            const int mv = decide<ASYNC, KI>(a, s_v[tid], s_c[tid], s_kv[tid], s_b[tid], bx != NO_CAND, unord_gain(o), bx);
            my_moves += mv;
            s_mv[tid] = mv;
        }
        __syncthreads();
        if (a.mark) {  // fused frontier: the same 8 positions per thread as phase 1
            const int p0 = tid * WIN_ITEMS;
            if (p0 < E) {
                int lo = 0, hi = nv;
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_loc[mid] <= p0) lo = mid; else hi = mid;
                }
                int sl = lo;
                for (int j = 0; j < WIN_ITEMS && p0 + j < E; ++j) {
                    const int p = p0 + j;
                    while (p >= s_loc[sl + 1]) ++sl;
                    if (s_mv[sl]) mark_nbr(a, __ldg(a.indices + s_start[sl] + (p - s_loc[sl])));
                }
            }
            __syncthreads();
        }
    }
    flush_moves(a, my_moves);
}

__global__ void k_window_starts(const int64_t* __restrict__ off, int64_t nb, int64_t nwin, int64_t* wstart) {
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w <= nwin; w += (int64_t)gridDim.x * blockDim.x) {
        // first list index whose prefix is >= w*W  (lower_bound over off[0..nb])
        const int64_t target = w * (int64_t)WIN_W;
        int64_t lo = 0, hi = nb + 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (off[mid] < target) lo = mid + 1; else hi = mid;
        }
        wstart[w] = w == nwin ? nb : (lo > nb ? nb : lo);
    }
}

struct DegOfList {
    const int64_t* indptr;
    const int32_t* list;
    int64_t n;
    __device__ __forceinline__ int64_t operator()(int64_t i) const {
        if (i >= n) return 0;
        const int32_t v = list[i];
        return indptr[v + 1] - indptr[v];
    }
};

// ===========================================================================
// large bin (hubs): vertices batched so that their global tables fit in L2.
// Per batch: insertion over LARGE_CHUNK-edge work items spread over all SMs,
// scoring over SCORE_CHUNK-slot work items (partial argmax per item), then a
// warp per vertex merges its partials and decides.  Batches are planned once
// on the host; no host synchronisation between batches.
// ===========================================================================
struct LargeBatch {
    const int32_t* list;       // batch vertices
    int64_t nL;
    const int64_t* cap_off;    // [nL+1] table slot offsets
    const int64_t* item_off;   // [nL+1] insertion work-item offsets
    const int64_t* sitem_off;  // [nL+1] scoring work-item offsets
    void* tab;                 // packed u64 slots, or int32 keys ...
    double* tabv;              // ... plus double sums (weighted)
    double* sc;                // [nL] S_c per vertex (own-cluster weight)
    double* pg;                // [scoring items] partial best gain
    int32_t* px;               // [scoring items] partial best cluster
};

template <bool FSUM>
__device__ __forceinline__ GlobalTable<FSUM> gtable(const LargeBatch& L, int64_t off) {
    if constexpr (FSUM) return GlobalTable<true>{static_cast<int32_t*>(L.tab) + off, L.tabv + off};
    else return GlobalTable<false>{static_cast<unsigned long long*>(L.tab) + off};
}

__device__ __forceinline__ int64_t owner_of(const int64_t* off, int64_t n, int64_t it) {
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (off[mid] <= it) lo = mid; else hi = mid;
    }
    return lo;
}

#ifndef LCC_LARGE_MINB
#define LCC_LARGE_MINB 4
#endif
template <class WT, bool ASYNC>
__global__ void __launch_bounds__(LARGE_THREADS, LCC_LARGE_MINB)
k_large_insert(BMArgs a, LargeBatch L, int64_t total_items) {
    constexpr int UL = 8;
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    for (int64_t it = blockIdx.x; it < total_items; it += gridDim.x) {
        const int64_t li = owner_of(L.item_off, L.nL, it);
        const int32_t v = L.list[li];
        const int64_t s = a.indptr[v], e_end = a.indptr[v + 1];
        const int64_t e0 = s + (it - L.item_off[li]) * LARGE_CHUNK;
        const int64_t e1 = min64(e0 + LARGE_CHUNK, e_end);
        const uint32_t cap = (uint32_t)(L.cap_off[li + 1] - L.cap_off[li]);
        const auto tab = gtable<WLoad<WT>::fsum>(L, L.cap_off[li]);
        const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
        double sc = 0.0;
        for (int64_t eb = e0 + threadIdx.x; eb < e1; eb += (int64_t)LARGE_THREADS * UL) {
            int32_t u[UL];
            typename WLoad<WT>::TW wv[UL];
#pragma unroll
            for (int j = 0; j < UL; ++j) {
                const int64_t e = eb + (int64_t)j * LARGE_THREADS;
                u[j] = e < e1 ? ld_stream_i32(a.indices + e, pol_stream) : -1;
                wv[j] = e < e1 ? WLoad<WT>::tw(a.w, e) : typename WLoad<WT>::TW(0);
            }
#pragma unroll
            for (int j = 0; j < UL; ++j) u[j] = u[j] >= 0 ? ldLabel<ASYNC>(a, u[j], pol_keep) : EMPTY_KEY;
            if constexpr (!WLoad<WT>::fsum) {
                // first probe of all UL keys issued back to back (UL device
                // CAS in flight per lane); collisions finish in the probe loop
                unsigned long long* T = static_cast<unsigned long long*>(L.tab) + L.cap_off[li];
                uint32_t h[UL];
                unsigned pending = 0;
#pragma unroll
                for (int j = 0; j < UL; ++j) {
                    h[j] = 0;
                    if (u[j] == EMPTY_KEY) continue;
                    if (u[j] == c) { sc += WLoad<WT>::f64(wv[j]); continue; }
                    h[j] = slot_of(u[j], cap);
                    pending |= 1u << j;
                }
                // every probe round issues the CAS of all pending keys back to
                // back, so a lane waits one L2 round trip per probe depth, not
                // per key
                while (pending) {
                    unsigned long long old[UL];
#pragma unroll
                    for (int j = 0; j < UL; ++j)
                        if (pending & (1u << j))
                            old[j] = atomicCAS(T + h[j], (unsigned long long)EMPTY64,
                                               ((unsigned long long)(uint32_t)u[j] << 32) | wv[j]);
#pragma unroll
                    for (int j = 0; j < UL; ++j) {
                        if (!(pending & (1u << j))) continue;
                        if (old[j] == EMPTY64) { pending &= ~(1u << j); continue; }
                        if ((int32_t)(old[j] >> 32) == u[j]) {
                            atomicAdd(T + h[j], (unsigned long long)wv[j]);
                            pending &= ~(1u << j);
                            continue;
                        }
                        h[j] = (h[j] + 1 == cap) ? 0 : h[j] + 1;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < UL; ++j) {
                    if (u[j] == EMPTY_KEY) continue;
                    if (u[j] == c) sc += wv[j];
                    else tab.insert(cap, u[j], wv[j]);
                }
            }
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) sc += __shfl_xor_sync(FULL, sc, d);
        if ((threadIdx.x & 31) == 0 && sc != 0.0) atomicAdd(L.sc + li, sc);
    }
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
    __syncthreads();
}

template <class WT, bool ASYNC, bool KI>
__global__ void __launch_bounds__(SCORE_THREADS)
k_large_score(BMArgs a, LargeBatch L, int64_t total_items) {
    constexpr int UL = 8;
    __shared__ double s_g[SCORE_THREADS / 32];
    __shared__ int32_t s_x[SCORE_THREADS / 32];
    const uint64_t pol_keep = policy_evict_last();
    for (int64_t it = blockIdx.x; it < total_items; it += gridDim.x) {
        const int64_t li = owner_of(L.sitem_off, L.nL, it);
        const int32_t v = L.list[li];
        const uint32_t cap = (uint32_t)(L.cap_off[li + 1] - L.cap_off[li]);
        const uint32_t q_begin = (uint32_t)((it - L.sitem_off[li]) * SCORE_CHUNK);
        const uint32_t q_end = (uint32_t)min64((int64_t)q_begin + SCORE_CHUNK, cap);
        const auto tab = gtable<WLoad<WT>::fsum>(L, L.cap_off[li]);
        const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
        const double kv = kval(a.k, v);
        const double Kc = ldMass<ASYNC, KI>(a, c, pol_keep);
        const double t = dmul(a.lam, kv);
        const double b = dadd(dsub(L.sc[li], dmul(t, Kc)), dmul(t, kv));
        double bg = -INFINITY;
        int32_t bx = NO_CAND;
        for (uint32_t q0 = q_begin + threadIdx.x; q0 < q_end; q0 += SCORE_THREADS * UL) {
            int32_t x[UL];
            double S[UL], Kx[UL];
#pragma unroll
            for (int j = 0; j < UL; ++j) {
                const uint32_t q = q0 + j * SCORE_THREADS;
                if (!(q < q_end && tab.read(q, x[j], S[j]))) x[j] = EMPTY_KEY;
            }
#pragma unroll
            for (int j = 0; j < UL; ++j) Kx[j] = x[j] != EMPTY_KEY ? ldMass<ASYNC, KI>(a, x[j], pol_keep) : 0.0;
#pragma unroll
            for (int j = 0; j < UL; ++j) {
                if (x[j] == EMPTY_KEY) continue;
                const double gq = dsub(dsub(S[j], dmul(t, Kx[j])), b);
                if (better(gq, x[j], bg, bx)) { bg = gq; bx = x[j]; }
            }
        }
        block_argmax<SCORE_THREADS>(bg, bx, s_g, s_x);
        if (threadIdx.x == 0) { L.pg[it] = bg; L.px[it] = bx; }
    }
}

template <class WT, bool ASYNC, bool KI>
__global__ void k_large_decide(BMArgs a, LargeBatch L) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint64_t pol_keep = policy_evict_last();
    unsigned long long my_moves = 0;
    for (int64_t li = gw; li < L.nL; li += nw) {
        double bg = -INFINITY;
        int32_t bx = NO_CAND;
        for (int64_t it = L.sitem_off[li] + lane; it < L.sitem_off[li + 1]; it += 32)
            if (better(L.pg[it], L.px[it], bg, bx)) { bg = L.pg[it]; bx = L.px[it]; }
        warp_argmax(bg, bx);
        if (lane == 0) {
            const int32_t v = L.list[li];
            const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
            const double kv = kval(a.k, v);
            const double Kc = ldMass<ASYNC, KI>(a, c, pol_keep);
            const double t = dmul(a.lam, kv);
            const double b = dadd(dsub(L.sc[li], dmul(t, Kc)), dmul(t, kv));
            double bS = NAN;  // the winner's S, for the commit-time check (the batch's table is intact)
            if (ASYNC && LCC_VALIDATE && bx != NO_CAND) {
                const uint32_t cap = (uint32_t)(L.cap_off[li + 1] - L.cap_off[li]);
                bS = gtable<WLoad<WT>::fsum>(L, L.cap_off[li]).find(cap, bx);
            }
            my_moves += decide<ASYNC, KI>(a, v, c, kv, b, bx != NO_CAND, bg, bx, bS);
        }
    }
    flush_moves(a, my_moves);
}

// fused frontier for hubs: every moved hub flags its neighbours, over the
// same LARGE_CHUNK-edge work items as the insertion
__global__ void __launch_bounds__(LARGE_THREADS)
k_large_mark(BMArgs a, LargeBatch L, int64_t total_items) {
    for (int64_t it = blockIdx.x; it < total_items; it += gridDim.x) {
        const int64_t li = owner_of(L.item_off, L.nL, it);
        const int32_t v = L.list[li];
        if (!a.moved[v]) continue;
        const int64_t s = a.indptr[v], e_end = a.indptr[v + 1];
        const int64_t e0 = s + (it - L.item_off[li]) * LARGE_CHUNK;
        const int64_t e1 = min64(e0 + LARGE_CHUNK, e_end);
#pragma unroll 4
        for (int64_t e = e0 + threadIdx.x; e < e1; e += LARGE_THREADS) mark_nbr(a, __ldg(a.indices + e));
    }
}


// ===========================================================================
// hub bin, bucket path (default for integer sums): the hub's neighbour labels
// are radix-partitioned by a hash of the label into buckets of ~HB_BE
// entries, then every bucket is aggregated by one CTA in a shared-memory
// table -- the same table as the group bins, so the hubs' per-edge work is
// shared-memory atomics instead of L2 CAS round trips on a 256 MB global
// table (and no table memset / write-back).
//   1. k_hub_scatter: LARGE_CHUNK-edge items (as the insert kernel); labels
//      gathered, the own-cluster weight summed, the rest counting-sorted by
//      bucket inside the item (shared-memory histogram + scan) and written
//      to the item's slot of `ent`, with per-item bucket offsets `ioff`.
//   2. k_hub_bucket: one CTA per (hub, bucket) walks the hub's items, inserts
//      its bucket's entries, scores its table -> partial (gain, id, S).
//   3. k_hub_decide: a warp per hub merges the partials and decides.
// A bucket whose entry count exceeds half the table is split into R passes
// by a second hash; a table that still fills sets an error flag (the round
// fails loudly; with murmur-hashed labels it does not happen).
// ===========================================================================
#ifndef LCC_HB_THREADS
#define LCC_HB_THREADS 256
#endif
constexpr int HB_THREADS = LCC_HB_THREADS;  // bucket CTA
constexpr int HS_THREADS = 256;             // scatter CTA
#ifndef LCC_HB_CAP
#define LCC_HB_CAP 4096
#endif
constexpr int HB_CAP = LCC_HB_CAP;      // table slots per bucket CTA
constexpr int HB_BE = HB_CAP / 2;       // target entries per bucket
constexpr int HB_MAXB = 256;            // buckets per hub (more -> larger buckets, multi-pass)
#ifndef LCC_HB_FLAT
#define LCC_HB_FLAT 1                   // bucket inserts flat over the bucket's entries
#endif
constexpr int HB_MAXIT = 1024;          // items per hub for the flat walk (2M edges)

template <class WT>
struct HubEntry {
    using T = typename std::conditional<WLoad<WT>::weighted, uint2, int32_t>::type;
    __device__ __forceinline__ static T make(int32_t x, uint32_t w) {
        if constexpr (WLoad<WT>::weighted) return make_uint2((uint32_t)x, w);
        else return x;
    }
    __device__ __forceinline__ static int32_t label(const T& e) {
        if constexpr (WLoad<WT>::weighted) return (int32_t)e.x;
        else return e;
    }
    __device__ __forceinline__ static uint32_t weight(const T& e) {
        if constexpr (WLoad<WT>::weighted) return e.y;
        else return 1u;
    }
};

struct HubPlan {
    const int32_t* list;      // hubs
    int64_t nL;
    const int64_t* item_off;  // [nL+1] LARGE_CHUNK items per hub
    const int64_t* boff;      // [nL+1] buckets per hub
    int stride;               // ioff entries per item (max buckets + 1)
    void* ent;                // [items * LARGE_CHUNK] bucketed entries
    int32_t* ioff;            // [items * stride] per-item bucket offsets
    double* sc;               // [nL] own-cluster weight
    double* pg;               // [buckets] partial best gain
    int32_t* px;              // [buckets] partial best cluster
    double* pS;               // [buckets] its S
    unsigned* overflow;
};

__device__ __forceinline__ uint32_t hub_bucket(int32_t x, uint32_t nb) {
    return (uint32_t)(((uint64_t)hash32((uint32_t)x) * nb) >> 32);
}
__device__ __forceinline__ uint32_t hub_pass(int32_t x, uint32_t R) {
    return hash32((uint32_t)x ^ 0x5bd1e995u) % R;
}

template <class WT, bool ASYNC>
__global__ void __launch_bounds__(HS_THREADS)
k_hub_scatter(BMArgs a, HubPlan P, int64_t total_items) {
    using E = HubEntry<WT>;
    using T = typename E::T;
    constexpr int PER = LARGE_CHUNK / HS_THREADS;  // 8 edges per thread
    __shared__ int s_hist[HB_MAXB + 1];
    __shared__ double s_red[HS_THREADS / 32];
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    const int tid = threadIdx.x;
    for (int64_t it = blockIdx.x; it < total_items; it += gridDim.x) {
        const int64_t li = owner_of(P.item_off, P.nL, it);
        const int32_t v = P.list[li];
        const int64_t s = a.indptr[v], e_end = a.indptr[v + 1];
        const int64_t e0 = s + (it - P.item_off[li]) * LARGE_CHUNK;
        const int64_t e1 = min64(e0 + LARGE_CHUNK, e_end);
        const uint32_t nb = (uint32_t)(P.boff[li + 1] - P.boff[li]);
        const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
        for (int b = tid; b <= (int)nb; b += HS_THREADS) s_hist[b] = 0;
        __syncthreads();
        int32_t x[PER];
        uint32_t w[PER];
        int bk[PER], rk[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int64_t e = e0 + (int64_t)j * HS_THREADS + tid;
            x[j] = e < e1 ? ld_stream_i32(a.indices + e, pol_stream) : -1;
            w[j] = e < e1 ? (uint32_t)WLoad<WT>::tw(a.w, e) : 0u;
        }
#pragma unroll
        for (int j = 0; j < PER; ++j) x[j] = x[j] >= 0 ? ldLabel<ASYNC>(a, x[j], pol_keep) : EMPTY_KEY;
        double sc = 0.0;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            bk[j] = -1;
            if (x[j] == EMPTY_KEY) continue;
            if (x[j] == c) { sc += u32_to_f64(w[j]); continue; }
            bk[j] = (int)hub_bucket(x[j], nb);
            rk[j] = atomicAdd(&s_hist[bk[j]], 1);
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) sc += __shfl_xor_sync(FULL, sc, d);
        if ((tid & 31) == 0) s_red[tid >> 5] = sc;
        __syncthreads();
        if (tid < 32) {  // exclusive scan of the bucket counts (nb <= HB_MAXB)
            int carry = 0;
            for (int b0 = 0; b0 <= (int)nb; b0 += 32) {
                const int b = b0 + tid;
                const int val = b < (int)nb ? s_hist[b] : 0;
                int incl = val;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const int y = __shfl_up_sync(FULL, incl, d);
                    if (tid >= d) incl += y;
                }
                if (b <= (int)nb) {
                    const int ex = carry + incl - val;
                    s_hist[b] = ex;
                    P.ioff[it * P.stride + b] = ex;
                }
                carry += __shfl_sync(FULL, incl, 31);
            }
            if (tid == 0) {
                double t = 0.0;
                for (int q = 0; q < HS_THREADS / 32; ++q) t += s_red[q];
                if (t != 0.0) atomicAdd(P.sc + li, t);
            }
        }
        __syncthreads();
        T* out = static_cast<T*>(P.ent) + it * LARGE_CHUNK;
#pragma unroll
        for (int j = 0; j < PER; ++j)
            if (bk[j] >= 0) out[s_hist[bk[j]] + rk[j]] = E::make(x[j], w[j]);
        __syncthreads();  // s_hist reused by the next item
    }
}

template <class WT, bool ASYNC, bool KI>
__global__ void __launch_bounds__(HB_THREADS)
k_hub_bucket(BMArgs a, HubPlan P, int64_t total_buckets) {
    using E = HubEntry<WT>;
    using T = typename E::T;
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ double s_g[HB_THREADS / 32], s_S[HB_THREADS / 32];
    __shared__ int32_t s_x[HB_THREADS / 32];
    __shared__ int64_t s_cnt;
    __shared__ int32_t s_pref[LCC_HB_FLAT ? HB_MAXIT + 1 : 1];
    SmemTable<false> tab;
    tab.init_cap(smem, HB_CAP);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    for (uint32_t q = tid; q < HB_CAP; q += HB_THREADS) tab.clear(q);
    const uint64_t pol_keep = policy_evict_last();
    for (int64_t gb = blockIdx.x; gb < total_buckets; gb += gridDim.x) {
        const int64_t li = owner_of(P.boff, P.nL, gb);
        const int b = (int)(gb - P.boff[li]);
        const int32_t v = P.list[li];
        const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
        const double kv = kval(a.k, v);
        const double t = dmul(a.lam, kv);
        const double Kc = ldMass<ASYNC, KI>(a, c, pol_keep);
        const double bb = dadd(dsub(P.sc[li], dmul(t, Kc)), dmul(t, kv));
        const int64_t i0 = P.item_off[li], i1 = P.item_off[li + 1];
        // entries of this bucket over the hub's items
        const int64_t nit = i1 - i0;
        const bool flat = LCC_HB_FLAT && nit <= HB_MAXIT;
        int64_t cnt;
        if (flat) {
            // per-item counts, prefix-summed in shared memory, so the inserts
            // run over the bucket's entries as one flat range (full lanes even
            // when a bucket holds a few entries of each of ~200 items)
            for (int64_t q = tid; q < nit; q += HB_THREADS) {
                const int64_t it = i0 + q;
                s_pref[q + 1] = P.ioff[it * P.stride + b + 1] - P.ioff[it * P.stride + b];
            }
            if (tid == 0) s_pref[0] = 0;
            __syncthreads();
            if (tid < 32) {
                int carry = 0;
                for (int64_t b0 = 1; b0 <= nit; b0 += 32) {
                    const int64_t q = b0 + lane;
                    const int val = q <= nit ? s_pref[q] : 0;
                    int incl = val;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const int y = __shfl_up_sync(FULL, incl, d);
                        if (lane >= d) incl += y;
                    }
                    if (q <= nit) s_pref[q] = carry + incl;
                    carry += __shfl_sync(FULL, incl, 31);
                }
            }
            __syncthreads();
            cnt = s_pref[nit];
        } else {
            if (tid == 0) s_cnt = 0;
            __syncthreads();
            int64_t mine = 0;
            for (int64_t it = i0 + tid; it < i1; it += HB_THREADS)
                mine += P.ioff[it * P.stride + b + 1] - P.ioff[it * P.stride + b];
            for (int d = 16; d; d >>= 1) mine += __shfl_xor_sync(FULL, mine, d);
            if (lane == 0 && mine) atomicAdd((unsigned long long*)&s_cnt, (unsigned long long)mine);
            __syncthreads();
            cnt = s_cnt;
        }
        const uint32_t R = (uint32_t)max64(1, (2 * cnt + HB_CAP - 1) / HB_CAP);
        const uint32_t cap = (uint32_t)min64(HB_CAP, (2 * ((cnt + R - 1) / R) + 31) & ~31LL);
        double bg = -INFINITY, bS = 0.0;
        int32_t bx = NO_CAND;
        for (uint32_t r = 0; r < R; ++r) {
            // insert: flat over the bucket's entries (item found by binary
            // search of the prefix), or warp w over items w, w+8, ...
            const int64_t nouter = flat ? 1 : nit;
            for (int64_t oi = flat ? 0 : wid; oi < nouter; oi += flat ? 1 : HB_THREADS / 32) {
                const int64_t it0 = i0 + oi;
                const int lo = flat ? 0 : P.ioff[it0 * P.stride + b];
                const int hi = flat ? (int)cnt : P.ioff[it0 * P.stride + b + 1];
                const int step = flat ? HB_THREADS : 32;
                for (int q = lo + (flat ? tid : lane); q < hi; q += step) {
                    T e;
                    if (flat) {
                        int l = 0, u = (int)nit;  // last item with s_pref[item] <= q
                        while (u - l > 1) {
                            const int m = (l + u) >> 1;
                            if (s_pref[m] <= q) l = m; else u = m;
                        }
                        const int64_t it = i0 + l;
                        e = static_cast<const T*>(P.ent)[it * LARGE_CHUNK + P.ioff[it * P.stride + b] + (q - s_pref[l])];
                    } else {
                        e = static_cast<const T*>(P.ent)[it0 * LARGE_CHUNK + q];
                    }
                    const int32_t x = E::label(e);
                    if (R > 1 && hub_pass(x, R) != r) continue;
                    uint32_t h = slot_of(x, cap);
                    uint32_t probes = 0;
                    int32_t prev;
                    while (true) {
                        asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(prev) : "r"(tab.keys + 4 * h), "r"(EMPTY_KEY), "r"(x) : "memory");
                        if (prev == EMPTY_KEY || prev == x) break;
                        h = (h + 1 == cap) ? 0 : h + 1;
                        if (++probes >= cap) { atomicOr(P.overflow, 1u); break; }
                    }
                    if (prev != EMPTY_KEY && prev != x) continue;  // overflow (reported)
                    const uint32_t inc = prev == EMPTY_KEY ? E::weight(e) - 1u : E::weight(e);
                    if (inc) asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(tab.cnts + 4 * h), "r"(inc) : "memory");
                }
            }
            __syncthreads();
            // score (and reset) the table
            for (uint32_t q0 = tid; q0 < cap; q0 += HB_THREADS * 4) {
                int32_t x[4];
                double S[4], Kx[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t q = q0 + j * HB_THREADS;
                    if (!(q < cap && tab.take(q, x[j], S[j]))) x[j] = EMPTY_KEY;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) Kx[j] = x[j] != EMPTY_KEY ? ldMass<ASYNC, KI>(a, x[j], pol_keep) : 0.0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (x[j] == EMPTY_KEY) continue;
                    const double gq = dsub(dsub(S[j], dmul(t, Kx[j])), bb);
                    if (better(gq, x[j], bg, bx)) { bg = gq; bx = x[j]; bS = S[j]; }
                }
            }
            __syncthreads();
        }
        warp_argmax(bg, bx, bS);
        if (lane == 0) { s_g[wid] = bg; s_x[wid] = bx; s_S[wid] = bS; }
        __syncthreads();
        if (tid == 0) {
            for (int q = 1; q < HB_THREADS / 32; ++q)
                if (better(s_g[q], s_x[q], bg, bx)) { bg = s_g[q]; bx = s_x[q]; bS = s_S[q]; }
            P.pg[gb] = bg;
            P.px[gb] = bx;
            P.pS[gb] = bS;
        }
        __syncthreads();
    }
}

template <class WT, bool ASYNC, bool KI>
__global__ void k_hub_decide(BMArgs a, HubPlan P) {
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    const uint64_t pol_keep = policy_evict_last();
    unsigned long long my_moves = 0;
    for (int64_t li = gw; li < P.nL; li += nw) {
        double bg = -INFINITY, bS = 0.0;
        int32_t bx = NO_CAND;
        for (int64_t q = P.boff[li] + lane; q < P.boff[li + 1]; q += 32)
            if (better(P.pg[q], P.px[q], bg, bx)) { bg = P.pg[q]; bx = P.px[q]; bS = P.pS[q]; }
        warp_argmax(bg, bx, bS);
        if (lane == 0) {
            const int32_t v = P.list[li];
            const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
            const double kv = kval(a.k, v);
            const double Kc = ldMass<ASYNC, KI>(a, c, pol_keep);
            const double t = dmul(a.lam, kv);
            const double b = dadd(dsub(P.sc[li], dmul(t, Kc)), dmul(t, kv));
            my_moves += decide<ASYNC, KI>(a, v, c, kv, b, bx != NO_CAND, bg, bx, bx != NO_CAND ? bS : NAN);
        }
    }
    flush_moves(a, my_moves);
}

// ===========================================================================
// hub bin, cluster path: one 8-CTA thread-block cluster per hub, its
// neighbour-cluster table spread over the 8 CTAs' shared memory (DSMEM,
// 8 x 24K slots: hubs up to ~98K edges).  Inserts are remote shared-memory
// CAS/RED (~215 cycles, no L2 traffic, the table never reaches DRAM); each
// CTA then scores its own slice from local shared memory.
//   1. edges split over the cluster; own-cluster weight summed per CTA;
//   2. barrier; every CTA reads the total S_c from CTA 0 -> b;
//   3. each CTA scores (and clears) its slice -> partial argmax to CTA 0;
//   4. barrier; CTA 0 decides; 5. barrier; movers' neighbours flagged.
// Unweighted / integer weights only (exact 32-bit sums).
// ===========================================================================
constexpr int HC_CL = 8;          // CTAs per cluster (portable maximum)
#ifndef LCC_HC_THREADS
#define LCC_HC_THREADS 1024
#endif
#ifndef LCC_HC_UL
#define LCC_HC_UL 2
#endif
constexpr int HC_THREADS = LCC_HC_THREADS;
constexpr int HC_SLICE = 24576;   // slots per CTA: 192 KB of keys + counts
constexpr int64_t HC_MAXDEG = (int64_t)HC_CL * HC_SLICE / 2;

__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_id() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_count() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_map(uint32_t smem_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(rank));
    return r;
}

template <class WT, bool ASYNC, bool KI>
__global__ void __launch_bounds__(HC_THREADS, 1)
k_hub_cluster(BMArgs a, const int32_t* __restrict__ hubs, int64_t nh) {
    static_assert(!WLoad<WT>::fsum, "cluster hub path: integer sums only");
    constexpr int UL = LCC_HC_UL;
    constexpr int NW = HC_THREADS / 32;
    using TW = typename WLoad<WT>::TW;
    extern __shared__ __align__(16) unsigned char smem[];
    uint32_t* keys = reinterpret_cast<uint32_t*>(smem);
    uint32_t* cnts = keys + HC_SLICE;
    __shared__ double s_red[NW];
    __shared__ int32_t s_redx[NW];
    __shared__ double s_sc[HC_CL];      // CTA 0: partial own-cluster weights
    __shared__ double s_pg[HC_CL];      // CTA 0: partial best gains
    __shared__ int32_t s_px[HC_CL];
    __shared__ int32_t s_moved;         // every CTA: did this hub move
    const uint32_t rank = cl_rank();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t keys_s = smem_u32(keys), cnts_s = smem_u32(cnts);
    for (int q = tid; q < HC_SLICE; q += HC_THREADS) {
        keys[q] = (uint32_t)EMPTY_KEY;
        cnts[q] = 0u;
    }
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();
    unsigned long long my_moves = 0;
    cl_sync();
    for (int64_t hi = cl_id(); hi < nh; hi += cl_count()) {
        const int32_t v = __ldg(hubs + hi);
        const int64_t s = __ldg(a.indptr + v), end = __ldg(a.indptr + v + 1);
        const uint32_t cap = (uint32_t)std::min<int64_t>((int64_t)HC_CL * HC_SLICE, (2 * (end - s) + 31) & ~31LL);
        const uint32_t per = (cap + HC_CL - 1) / HC_CL;
        const int32_t c = ldLabel<ASYNC>(a, v, pol_keep);
        // ---- 1. inserts (remote shared-memory atomics)
        double sc = 0.0;
        for (int64_t e0 = s + (int64_t)rank * HC_THREADS + tid; e0 < end; e0 += (int64_t)HC_CL * HC_THREADS * UL) {
            int32_t u[UL];
            TW wv[UL];
#pragma unroll
            for (int j = 0; j < UL; ++j) {
                const int64_t e = e0 + (int64_t)j * HC_CL * HC_THREADS;
                u[j] = e < end ? ld_stream_i32(a.indices + e, pol_stream) : -1;
                wv[j] = e < end ? WLoad<WT>::tw(a.w, e) : TW(0);
            }
#pragma unroll
            for (int j = 0; j < UL; ++j) u[j] = u[j] >= 0 ? ldLabel<ASYNC>(a, u[j], pol_keep) : EMPTY_KEY;
            uint32_t h[UL];
            unsigned pending = 0;
#pragma unroll
            for (int j = 0; j < UL; ++j) {
                h[j] = 0;
                if (u[j] == EMPTY_KEY) continue;
                if (u[j] == c) { sc += WLoad<WT>::f64(wv[j]); continue; }
                h[j] = slot_of(u[j], cap);
                pending |= 1u << j;
            }
            while (pending) {
                uint32_t prev[UL], addr[UL];
#pragma unroll
                for (int j = 0; j < UL; ++j) {
                    if (!(pending & (1u << j))) continue;
                    const uint32_t o = h[j] / per, l = h[j] - o * per;
                    addr[j] = cl_map(keys_s + 4 * l, o);
                    asm volatile("atom.shared::cluster.cas.b32 %0, [%1], %2, %3;"
                                 : "=r"(prev[j]) : "r"(addr[j]), "r"((uint32_t)EMPTY_KEY), "r"((uint32_t)u[j]) : "memory");
                }
#pragma unroll
                for (int j = 0; j < UL; ++j) {
                    if (!(pending & (1u << j))) continue;
                    if (prev[j] == (uint32_t)EMPTY_KEY || prev[j] == (uint32_t)u[j]) {
                        // counts sit HC_SLICE words after the key in the same CTA
                        asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(addr[j] + 4 * HC_SLICE), "r"((uint32_t)wv[j])
                                     : "memory");
                        pending &= ~(1u << j);
                    } else {
                        h[j] = (h[j] + 1 == cap) ? 0 : h[j] + 1;
                    }
                }
            }
        }
        // own-cluster weight: block sum -> CTA 0
#pragma unroll
        for (int d = 16; d; d >>= 1) sc += __shfl_xor_sync(FULL, sc, d);
        if (lane == 0) s_red[wid] = sc;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < NW; ++w) t += s_red[w];
            const uint32_t dst = cl_map(smem_u32(&s_sc[rank]), 0);
            asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dst), "d"(t) : "memory");
        }
        cl_sync();  // inserts complete, partial S_c published
        // ---- 2. b from the total S_c (summed in rank order on every CTA)
        double sct = 0.0;
        for (int r = 0; r < HC_CL; ++r) {
            double x;
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(x) : "r"(cl_map(smem_u32(&s_sc[r]), 0)) : "memory");
            sct += x;
        }
        const double kv = kval(a.k, v);
        const double Kc = ldMass<ASYNC, KI>(a, c, pol_keep);
        const double t = dmul(a.lam, kv);
        const double b = dadd(dsub(sct, dmul(t, Kc)), dmul(t, kv));
        // ---- 3. score (and clear) the local slice
        double bg = -INFINITY;
        int32_t bx = NO_CAND;
        const uint32_t lo = rank * per, hiq = std::min<uint32_t>(cap, lo + per);
        for (uint32_t q0 = tid; lo + q0 < hiq; q0 += HC_THREADS * UL) {
            int32_t x[UL];
            double S[UL], Kx[UL];
#pragma unroll
            for (int j = 0; j < UL; ++j) {
                const uint32_t q = q0 + j * HC_THREADS;
                x[j] = EMPTY_KEY;
                if (lo + q < hiq) {
                    const uint32_t kq = keys[q];
                    if (kq != (uint32_t)EMPTY_KEY) {
                        x[j] = (int32_t)kq;
                        S[j] = u32_to_f64(cnts[q]);
                        keys[q] = (uint32_t)EMPTY_KEY;
                        cnts[q] = 0u;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < UL; ++j) Kx[j] = x[j] != EMPTY_KEY ? ldMass<ASYNC, KI>(a, x[j], pol_keep) : 0.0;
#pragma unroll
            for (int j = 0; j < UL; ++j) {
                if (x[j] == EMPTY_KEY) continue;
                const double gq = dsub(dsub(S[j], dmul(t, Kx[j])), b);
                if (better(gq, x[j], bg, bx)) { bg = gq; bx = x[j]; }
            }
        }
        warp_argmax(bg, bx);
        if (lane == 0) { s_red[wid] = bg; s_redx[wid] = bx; }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < NW; ++w)
                if (better(s_red[w], s_redx[w], bg, bx)) { bg = s_red[w]; bx = s_redx[w]; }
            asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(cl_map(smem_u32(&s_pg[rank]), 0)), "d"(bg) : "memory");
            asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cl_map(smem_u32(&s_px[rank]), 0)), "r"(bx) : "memory");
        }
        cl_sync();  // partial argmaxes at CTA 0, every slice cleared
        // ---- 4. decide (CTA 0) and tell the cluster
        if (rank == 0 && tid == 0) {
            double g = s_pg[0];
            int32_t x = s_px[0];
            for (int r = 1; r < HC_CL; ++r)
                if (better(s_pg[r], s_px[r], g, x)) { g = s_pg[r]; x = s_px[r]; }
            const int mv = decide<ASYNC, KI>(a, v, c, kv, b, x != NO_CAND, g, x);
            my_moves += mv;
            for (int r = 0; r < HC_CL; ++r)
                asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(cl_map(smem_u32(&s_moved), r)), "r"(mv) : "memory");
        }
        if (a.mark) {
            cl_sync();
            if (s_moved) {
                for (int64_t e = s + (int64_t)rank * HC_THREADS + tid; e < end; e += (int64_t)HC_CL * HC_THREADS)
                    mark_nbr(a, __ldg(a.indices + e));
            }
        }
        cl_sync();  // s_moved / s_sc / s_pg free for the next hub
    }
    flush_moves(a, my_moves);
}

// ===========================================================================
// degree-bin partition (one pass, block-aggregated reservations)
// ===========================================================================
constexpr int NBINS = 11;
struct BinEdges {
    int64_t hi[NBINS];  // bin b holds hi[b-1] < deg <= hi[b]  (hi[-1] = -1)
};

// Stable partition (frontier order preserved inside every bin, so sorted
// frontiers give id-ordered bins): pass 1 counts per (bin, tile), an
// exclusive scan gives every (bin, tile) its output offset, pass 2 scatters
// with warp-ballot ranks.
constexpr int BIN_THREADS = 256;
constexpr int BIN_ROUNDS = 8;
constexpr int BIN_TILE = BIN_THREADS * BIN_ROUNDS;

__device__ __forceinline__ int bin_of(int64_t d, const BinEdges& be) {
    int bin = 0;
#pragma unroll
    for (int b = 0; b < NBINS - 1; ++b) bin += d > be.hi[b] ? 1 : 0;
    return bin;
}

__global__ void __launch_bounds__(BIN_THREADS)
k_bin_count(const int64_t* __restrict__ indptr, const int32_t* __restrict__ frontier, int64_t nF, BinEdges be,
            int64_t ntiles, int64_t* tile_counts, unsigned long long* edges) {
    __shared__ unsigned s_cnt[NBINS];
    const int64_t tile = blockIdx.x;
    if (threadIdx.x < NBINS) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    unsigned long long my_edges = 0;
    for (int r = 0; r < BIN_ROUNDS; ++r) {
        const int64_t i = tile * BIN_TILE + (int64_t)r * BIN_THREADS + threadIdx.x;
        if (i < nF) {
            const int32_t v = frontier ? frontier[i] : (int32_t)i;
            const int64_t d = indptr[v + 1] - indptr[v];
            my_edges += (unsigned long long)d;
            atomicAdd(&s_cnt[bin_of(d, be)], 1u);
        }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) my_edges += __shfl_xor_sync(FULL, my_edges, d);
    if ((threadIdx.x & 31) == 0 && my_edges) atomicAdd(edges, my_edges);
    __syncthreads();
    if (threadIdx.x < NBINS) tile_counts[(int64_t)threadIdx.x * ntiles + tile] = s_cnt[threadIdx.x];
}

__global__ void __launch_bounds__(BIN_THREADS)
k_bin_scatter(const int64_t* __restrict__ indptr, const int32_t* __restrict__ frontier, int64_t nF, BinEdges be,
              int64_t ntiles, const int64_t* __restrict__ tile_base, int32_t* __restrict__ out) {
    constexpr int W = BIN_THREADS / 32;
    __shared__ unsigned s_wc[W][NBINS];
    __shared__ int64_t s_run[NBINS];
    const int64_t tile = blockIdx.x;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x < NBINS) s_run[threadIdx.x] = tile_base[(int64_t)threadIdx.x * ntiles + tile];
    for (int r = 0; r < BIN_ROUNDS; ++r) {
        const int64_t i = tile * BIN_TILE + (int64_t)r * BIN_THREADS + threadIdx.x;
        int bin = -1;
        int32_t v = 0;
        if (i < nF) {
            v = frontier ? frontier[i] : (int32_t)i;
            bin = bin_of(indptr[v + 1] - indptr[v], be);
        }
        unsigned rank = 0;
#pragma unroll
        for (int b = 0; b < NBINS; ++b) {
            const unsigned m = __ballot_sync(FULL, bin == b);
            if (bin == b) rank = __popc(m & ((1u << lane) - 1u));
            if (lane == 0) s_wc[w][b] = __popc(m);
        }
        __syncthreads();
        if (bin >= 0) {
            int64_t pos = s_run[bin] + rank;
            for (int ww = 0; ww < w; ++ww) pos += s_wc[ww][bin];
            out[pos] = v;  // bins are contiguous, in bin order, in one array
        }
        __syncthreads();
        if (threadIdx.x < NBINS) {
            unsigned tot = 0;
            for (int ww = 0; ww < W; ++ww) tot += s_wc[ww][threadIdx.x];
            s_run[threadIdx.x] += tot;
        }
        __syncthreads();
    }
}

__global__ void k_degrees_of(const int64_t* __restrict__ indptr, const int32_t* __restrict__ list, int64_t n,
                             int64_t* out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = list[i];
        out[i] = indptr[v + 1] - indptr[v];
    }
}

// ---- integer masses ------------------------------------------------------
// Every BASELINE config has integer k (k = 1, or k = unweighted degree), so
// every cluster mass K_c is an integer.  When a round covers a large part of
// the graph, K is copied into a uint32 image for the round: the per-candidate
// mass gathers then read 4 instead of 8 bytes from an array half the size
// (config 4: labels 67 MB + masses 67 MB stay L2-resident, against 67 + 134
// MB).  u32 -> f64 is exact, so every gain is bit-identical.  The copy checks
// integrality (K and k), non-negativity and sum(K) < 2^31 (no transient sum
// can wrap); any failure keeps the fp64 kernels for the round.
__global__ void k_mass_to_u32(const double* __restrict__ K, int64_t klen, const double* __restrict__ k, int64_t n,
                              uint32_t* __restrict__ Ki, unsigned long long* sum, unsigned* bad, unsigned* maxv) {
    unsigned long long my = 0;
    unsigned mx = 0;  // largest mass / vertex weight seen (packed rounds need them small)
    bool ok = true;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < klen; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = K[i];
        const bool good = x >= 0.0 && x < 2147483648.0 && x == floor(x);
        ok &= good;
        const uint32_t u = good ? (uint32_t)x : 0u;
        Ki[KS * i] = u;
        my += u;
        mx = max(mx, u);
        if (k && i < n) {
            const double kv = k[i];
            const bool kgood = kv >= 0.0 && kv < 2147483648.0 && kv == floor(kv);
            ok &= kgood;
            if (kgood) mx = max(mx, (unsigned)kv);
        }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) my += __shfl_xor_sync(FULL, my, d);
#pragma unroll
    for (int d = 16; d; d >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, d));
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(maxv, mx);
    if ((threadIdx.x & 31) == 0 && my) atomicAdd(sum, my);
    if (__any_sync(FULL, !ok) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}
__global__ void k_mass_from_u32(const uint32_t* __restrict__ Ki, int64_t klen, double* __restrict__ K) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < klen; i += (int64_t)gridDim.x * blockDim.x)
        K[i] = u32_to_f64(Ki[KS * i]);
}
// LK[v] = C[v] | Ki[C[v]] << 32: the packed word the group bins gather
__global__ void k_pack_lk(const int32_t* __restrict__ C, const uint32_t* __restrict__ Ki, int64_t n,
                          unsigned long long* __restrict__ LK) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = C[v];
        LK[v] = (unsigned long long)(uint32_t)c | ((unsigned long long)Ki[KS * c] << 32);
    }
}
// interleaved labels: CK[2v] = C[v] before the round, C[v] = CK[2v] after an async one
__global__ void k_labels_in(const int32_t* __restrict__ C, int64_t n, int32_t* __restrict__ CK) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        CK[2 * v] = C[v];
}
__global__ void k_labels_out(const int32_t* __restrict__ CK, int64_t n, int32_t* __restrict__ C) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        C[v] = CK[2 * v];
}

// packed rounds: W[i] = (label of vertex i, i < n) | (mass of cluster i) << lb
__global__ void k_pack32(const int32_t* __restrict__ C, const uint32_t* __restrict__ Ki, int64_t n, int64_t klen, int lb,
                         uint32_t* __restrict__ W) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < klen; i += (int64_t)gridDim.x * blockDim.x)
        W[i] = (i < n ? (uint32_t)C[i] : 0u) | (Ki[KS * i] << lb);
}
// codes of a packed round (BMArgs::code): one thread per 8 vertices; *nvalid counts the set codes
__global__ void k_codes(const int32_t* __restrict__ C, const uint32_t* __restrict__ Ki, int64_t n, unsigned* __restrict__ code,
                        unsigned long long* nvalid) {
    const int64_t nw = (n + 7) / 8;
    unsigned long long mine = 0;
    for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nw; w += (int64_t)gridDim.x * blockDim.x) {
        unsigned word = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int64_t i = 8 * w + j;
            if (i < n) {
                const uint32_t m = Ki[KS * i];
                if (C[i] == (int32_t)i && m >= 1u && m <= 15u) {
                    word |= m << (4 * j);
                    ++mine;
                }
            }
        }
        code[w] = word;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) mine += __shfl_xor_sync(FULL, mine, d);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(nvalid, mine);
}
__global__ void k_unpack32(const uint32_t* __restrict__ W, int64_t n, int64_t klen, int lb, int32_t* __restrict__ C,
                           double* __restrict__ K) {
    const uint32_t lm = (1u << lb) - 1u;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < klen; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t w = W[i];
        if (i < n) C[i] = (int32_t)(w & lm);
        K[i] = u32_to_f64(w >> lb);
    }
}

template <class K>
void set_smem(K kernel, int bytes) {
    LCC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

template <class WT, bool ASYNC, bool KI, int GW, int CAP, int GROUPS, int U, int MINB = 1>
void launch_group(const BMArgs& a, const int32_t* list, int64_t lo, int64_t hi, cudaStream_t s) {
    if (hi <= lo) return;
    constexpr int THREADS = GW * 32 * GROUPS;
    constexpr int SMEM = (int)group_smem_bytes<WT, ASYNC, KI, CAP, GROUPS>();
    static int occ = 0;
    if (!occ) {
        set_smem(k_group<WT, ASYNC, KI, GW, CAP, GROUPS, U, MINB>, SMEM);
        LCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_group<WT, ASYNC, KI, GW, CAP, GROUPS, U, MINB>, THREADS, SMEM));
        occ = std::max(occ, 1);
    }
    const int64_t blocks_needed = (hi - lo + GROUPS - 1) / GROUPS;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(blocks_needed, (int64_t)num_sms() * occ));
    k_group<WT, ASYNC, KI, GW, CAP, GROUPS, U, MINB><<<grid, THREADS, SMEM, s>>>(a, list, lo, hi);
    LCC_LAUNCH_CHECK();
}

constexpr int B5_CAP = 16384;
constexpr int64_t MED_MAX = (B5_CAP * 5) / 8;      // 10240: load factor <= 0.625
#ifndef LCC_LARGE_TABLE_MB
#define LCC_LARGE_TABLE_MB 256
#endif
constexpr int64_t LARGE_TABLE_BYTES = (int64_t)LCC_LARGE_TABLE_MB << 20;  // per batch: stays L2-resident

// bin -> kernel shape.  Shared memory per group = CAP * (4 key + 4|8 value +
// 2 slot-list) bytes; GROUPS chosen so 2-3 CTAs fit per SM.
template <class WT, bool ASYNC, bool KI>
void launch_bin(int bin, const BMArgs& a, const int32_t* list, int64_t lo, int64_t hi, cudaStream_t s) {
    // LCC_VARIANT (env, tuning only) selects alternative group shapes
    const char* ev = getenv("LCC_VARIANT");
    const int var = ev ? atoi(ev) : 0;
    switch (bin) {  //                         GW  CAP    GROUPS U
        case 2: launch_group<WT, ASYNC, KI, 1, 256, 8, 4, 6>(a, list, lo, hi, s); break;   //  ..128      warp
        case 3: launch_group<WT, ASYNC, KI, 1, 1024, 8, 8, 3>(a, list, lo, hi, s); break;  //  ..512      warp
        case 4:  // ..1023: 2048-slot tables, 4 groups of 4 warps per CTA (measured +3.3% vs 4096 slots x 2)
            if (var == 8) launch_group<WT, ASYNC, KI, 2, 2048, 4, 8, 4>(a, list, lo, hi, s);
            else launch_group<WT, ASYNC, KI, 4, 2048, 4, 4, 2>(a, list, lo, hi, s);
            break;
        case 5:
            if (var == 3) launch_group<WT, ASYNC, KI, 8, 4096, 1, 8>(a, list, lo, hi, s);
            else launch_group<WT, ASYNC, KI, 4, 4096, 2, 8, 3>(a, list, lo, hi, s);        //  ..2048     4 warps
            break;
        case 6:
            if (var == 1) launch_group<WT, ASYNC, KI, 16, 8192, 1, 8>(a, list, lo, hi, s);
            else if (var == 4) launch_group<WT, ASYNC, KI, 4, 8192, 1, 8, 3>(a, list, lo, hi, s);
            else launch_group<WT, ASYNC, KI, 8, 8192, 1, 4>(a, list, lo, hi, s);           //  ..4096     8 warps
            break;
        case 7:
            if (var == 1) launch_group<WT, ASYNC, KI, 16, B5_CAP, 1, 8>(a, list, lo, hi, s);
            else if (var == 4) launch_group<WT, ASYNC, KI, 8, B5_CAP, 1, 4, 1>(a, list, lo, hi, s);
            else launch_group<WT, ASYNC, KI, 32, B5_CAP, 1, 4>(a, list, lo, hi, s);        //  ..10240    32 warps
            break;
        default: break;
    }
}

// window bin: degree prefix over the bin list -> window starts
struct WindowPlan {
    Buf<int64_t> off, wstart;
    int64_t nwin = 0;
};
inline void plan_windows(const int64_t* indptr, const int32_t* list, int64_t nb, WindowPlan& P, cudaStream_t s) {
    P.off.alloc(nb + 1, s);
    cub::TransformInputIterator<int64_t, DegOfList, cub::CountingInputIterator<int64_t>> degs(
        cub::CountingInputIterator<int64_t>(0), DegOfList{indptr, list, nb});
    exclusive_sum(degs, P.off.get(), nb + 1, s);
    int64_t total = 0;
    LCC_CUDA(cudaMemcpyAsync(&total, P.off.get() + nb, sizeof(total), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    P.nwin = (total + WIN_W - 1) / WIN_W;
    if (P.nwin < 1) P.nwin = 1;
    P.wstart.alloc(P.nwin + 1, s);
    k_window_starts<<<grid_for(P.nwin + 1, 256), 256, 0, s>>>(P.off.get(), nb, P.nwin, P.wstart.get());
    LCC_LAUNCH_CHECK();
}

template <class WT, bool ASYNC, bool KI>
void launch_window(const BMArgs& a, const int32_t* list, const WindowPlan& P, int64_t w0, int64_t w1, cudaStream_t s) {
    if (w1 <= w0) return;
    constexpr int SMEM = (int)window_smem_bytes<WLoad<WT>::fsum>();
    static int occ = 0;
    if (!occ) {
        set_smem(k_window<WT, ASYNC, KI>, SMEM);
        LCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_window<WT, ASYNC, KI>, WIN_THREADS, SMEM));
        occ = std::max(occ, 1);
    }
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(w1 - w0, (int64_t)num_sms() * occ));
    k_window<WT, ASYNC, KI><<<grid, WIN_THREADS, SMEM, s>>>(a, list, P.off.get(), P.wstart.get(), w0, w1);
    LCC_LAUNCH_CHECK();
}

inline int64_t large_cap(int64_t deg) { return (2 * deg + 31) & ~31LL; }

template <class WT, bool ASYNC, bool KI>
void launch_hub_cluster(const BMArgs& a, const int32_t* hubs, int64_t nh, cudaStream_t s) {
    constexpr int SMEM = HC_SLICE * 8;
    static int max_clusters = 0;
    auto kern = k_hub_cluster<WT, ASYNC, KI>;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = HC_CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(HC_THREADS);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (!max_clusters) {
        set_smem(kern, SMEM);
        cfg.gridDim = dim3(HC_CL * 64);
        LCC_CUDA(cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg));
        max_clusters = std::max(max_clusters, 1);
    }
    const int nc = (int)std::min<int64_t>(nh, max_clusters);
    cfg.gridDim = dim3(HC_CL * nc);
    LCC_CUDA(cudaLaunchKernelEx(&cfg, kern, a, hubs, nh));
    LCC_LAUNCH_CHECK();
}

// hub bucket path (integer sums): plan on the host, three kernels + the mark
template <class WT, bool ASYNC, bool KI>
void run_hub_buckets(const BMArgs& a, const int32_t* large, const std::vector<int64_t>& deg, unsigned* ovf,
                     cudaStream_t s) {
    using T = typename HubEntry<WT>::T;
    const int64_t nL = (int64_t)deg.size();
    std::vector<int64_t> h(2 * (nL + 1));
    int64_t* item_off = h.data();
    int64_t* boff = h.data() + nL + 1;
    item_off[0] = boff[0] = 0;
    int maxb = 1;
    for (int64_t i = 0; i < nL; ++i) {
        const int64_t nb = std::min<int64_t>(HB_MAXB, std::max<int64_t>(1, (deg[i] + HB_BE - 1) / HB_BE));
        maxb = std::max<int>(maxb, (int)nb);
        item_off[i + 1] = item_off[i] + (deg[i] + LARGE_CHUNK - 1) / LARGE_CHUNK;
        boff[i + 1] = boff[i] + nb;
    }
    const int64_t items = item_off[nL], buckets = boff[nL];
    const int stride = maxb + 1;
    Buf<int64_t> offs(h.size(), s);
    LCC_CUDA(cudaMemcpyAsync(offs.get(), h.data(), sizeof(int64_t) * h.size(), cudaMemcpyHostToDevice, s));
    Buf<T> ent(items * LARGE_CHUNK, s);
    Buf<int32_t> ioff(items * stride, s);
    Buf<double> sc(nL, s), pg(buckets, s), pS(buckets, s);
    Buf<int32_t> px(buckets, s);
    LCC_CUDA(cudaMemsetAsync(sc.get(), 0, sizeof(double) * nL, s));
    HubPlan P{large, nL, offs.get(), offs.get() + nL + 1, stride, ent.get(), ioff.get(), sc.get(), pg.get(), px.get(),
              pS.get(), ovf};
    k_hub_scatter<WT, ASYNC><<<grid_for(items * HS_THREADS, HS_THREADS, 8), HS_THREADS, 0, s>>>(a, P, items);
    LCC_LAUNCH_CHECK();
    constexpr int SMEM = HB_CAP * SmemTable<false>::bytes_per_slot;
    static int occ = 0;
    if (!occ) {
        set_smem(k_hub_bucket<WT, ASYNC, KI>, SMEM);
        LCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_hub_bucket<WT, ASYNC, KI>, HB_THREADS, SMEM));
        occ = std::max(occ, 1);
    }
    const unsigned gridb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(buckets, (int64_t)num_sms() * occ));
    k_hub_bucket<WT, ASYNC, KI><<<gridb, HB_THREADS, SMEM, s>>>(a, P, buckets);
    LCC_LAUNCH_CHECK();
    k_hub_decide<WT, ASYNC, KI><<<grid_for(nL * 32, 256), 256, 0, s>>>(a, P);
    LCC_LAUNCH_CHECK();
    if (a.mark) {
        LargeBatch L{large, nL, nullptr, offs.get(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        k_large_mark<<<grid_for(items * LARGE_THREADS, LARGE_THREADS, 8), LARGE_THREADS, 0, s>>>(a, L, items);
        LCC_LAUNCH_CHECK();
    }
}

template <class WT, bool ASYNC, bool KI>
void run_large(const BMArgs& a, const lcc_graph& g, const int32_t* large_in, int64_t nL_in, unsigned* ovf,
               cudaStream_t s) {
    constexpr bool WEIGHTED = WLoad<WT>::fsum;  // float sums: key + f64 value tables
    Buf<int64_t> ddeg(nL_in, s);
    k_degrees_of<<<grid_for(nL_in, 256), 256, 0, s>>>(g.indptr, large_in, nL_in, ddeg.get());
    LCC_LAUNCH_CHECK();
    std::vector<int64_t> deg_in(nL_in);
    std::vector<int32_t> ids(nL_in);
    LCC_CUDA(cudaMemcpyAsync(deg_in.data(), ddeg.get(), sizeof(int64_t) * nL_in, cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaMemcpyAsync(ids.data(), large_in, sizeof(int32_t) * nL_in, cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    // LCC_HUB_CLUSTER=1: hubs whose table fits one 8-CTA cluster's shared
    // memory take the DSMEM path (integer sums).  Off by default: measured
    // 35.6 vs 39.1 Gedges/s on config 4 (one hub per cluster at a time leaves
    // the SMs underfed; the L2 tables process every hub's edges at once).
    std::vector<int32_t> hc, l2;
    std::vector<int64_t> deg;
    const char* ehc = getenv("LCC_HUB_CLUSTER");
    const bool use_hc = !WEIGHTED && ehc && ehc[0] == '1';
    for (int64_t i = 0; i < nL_in; ++i) {
        if (use_hc && deg_in[i] <= HC_MAXDEG) {
            hc.push_back(ids[i]);
        } else {
            l2.push_back(ids[i]);
            deg.push_back(deg_in[i]);
        }
    }
    Buf<int32_t> dlists(std::max<size_t>(hc.size() + l2.size(), 1), s);
    if (!hc.empty())
        LCC_CUDA(cudaMemcpyAsync(dlists.get(), hc.data(), sizeof(int32_t) * hc.size(), cudaMemcpyHostToDevice, s));
    if (!l2.empty())
        LCC_CUDA(cudaMemcpyAsync(dlists.get() + hc.size(), l2.data(), sizeof(int32_t) * l2.size(),
                                 cudaMemcpyHostToDevice, s));
    if constexpr (!WEIGHTED) {
        if (!hc.empty()) launch_hub_cluster<WT, ASYNC, KI>(a, dlists.get(), (int64_t)hc.size(), s);
    }
    const int32_t* large = dlists.get() + hc.size();
    const int64_t nL = (int64_t)l2.size();
    if (nL == 0) return;
    const char* ehb = getenv("LCC_HUB_BUCKETS");
    if constexpr (!WEIGHTED) {
        if (!(ehb && ehb[0] == '0')) {
            run_hub_buckets<WT, ASYNC, KI>(a, large, deg, ovf, s);
            return;
        }
    }
    const int64_t slot_bytes = GlobalTable<WEIGHTED>::bytes_per_slot;
    int64_t maxcap = 0;
    for (int64_t d : deg) maxcap = std::max<int64_t>(maxcap, large_cap(d));
    const int64_t table_slots = std::max<int64_t>(LARGE_TABLE_BYTES / slot_bytes, maxcap);
    // plan every batch: per-batch relative offsets, concatenated
    struct B { int64_t b0, nb, slots, items, sitems, off; };
    std::vector<B> batches;
    std::vector<int64_t> h;  // for each batch: cap_off[nb+1], item_off[nb+1], sitem_off[nb+1]
    int64_t max_sitems = 0;
    for (int64_t b0 = 0; b0 < nL;) {
        int64_t b1 = b0, slots = 0, items = 0, sitems = 0;
        const size_t base = h.size();
        h.resize(base + 3 * (nL - b0 + 1));
        std::vector<int64_t> co, io, so;
        while (b1 < nL) {
            const int64_t cap = large_cap(deg[b1]);
            if (b1 > b0 && slots + cap > table_slots) break;
            co.push_back(slots); io.push_back(items); so.push_back(sitems);
            slots += cap;
            items += (deg[b1] + LARGE_CHUNK - 1) / LARGE_CHUNK;
            sitems += (cap + SCORE_CHUNK - 1) / SCORE_CHUNK;
            ++b1;
        }
        co.push_back(slots); io.push_back(items); so.push_back(sitems);
        const int64_t nb = b1 - b0;
        h.resize(base);
        h.insert(h.end(), co.begin(), co.end());
        h.insert(h.end(), io.begin(), io.end());
        h.insert(h.end(), so.begin(), so.end());
        batches.push_back(B{b0, nb, slots, items, sitems, (int64_t)base});
        max_sitems = std::max(max_sitems, sitems);
        b0 = b1;
    }
    Buf<int64_t> offs(h.size(), s);
    LCC_CUDA(cudaMemcpyAsync(offs.get(), h.data(), sizeof(int64_t) * h.size(), cudaMemcpyHostToDevice, s));
    Buf<unsigned long long> tab(WEIGHTED ? (table_slots + 1) / 2 : table_slots, s);  // u64 slots or i32 keys
    Buf<double> tabv(WEIGHTED ? table_slots : 0, s);
    Buf<double> sc(nL, s);
    Buf<double> pg(max_sitems, s);
    Buf<int32_t> px(max_sitems, s);
    LCC_CUDA(cudaMemsetAsync(sc.get(), 0, sizeof(double) * nL, s));
    for (const B& bt : batches) {
        const int64_t* o = offs.get() + bt.off;
        LargeBatch L{large + bt.b0, bt.nb, o, o + (bt.nb + 1), o + 2 * (bt.nb + 1), tab.get(), tabv.get(),
                     sc.get() + bt.b0, pg.get(), px.get()};
        if (WEIGHTED) {
            LCC_CUDA(cudaMemsetAsync(tab.get(), 0xff, sizeof(int32_t) * bt.slots, s));
            LCC_CUDA(cudaMemsetAsync(tabv.get(), 0, sizeof(double) * bt.slots, s));
        } else {
            LCC_CUDA(cudaMemsetAsync(tab.get(), 0xff, sizeof(unsigned long long) * bt.slots, s));
        }
        k_large_insert<WT, ASYNC><<<grid_for(bt.items * LARGE_THREADS, LARGE_THREADS, 8), LARGE_THREADS, 0, s>>>(a, L, bt.items);
        LCC_LAUNCH_CHECK();
        k_large_score<WT, ASYNC, KI><<<grid_for(bt.sitems * SCORE_THREADS, SCORE_THREADS, 4), SCORE_THREADS, 0, s>>>(a, L, bt.sitems);
        LCC_LAUNCH_CHECK();
        k_large_decide<WT, ASYNC, KI><<<grid_for(bt.nb * 32, 256), 256, 0, s>>>(a, L);
        LCC_LAUNCH_CHECK();
        if (a.mark) {
            k_large_mark<<<grid_for(bt.items * LARGE_THREADS, LARGE_THREADS, 8), LARGE_THREADS, 0, s>>>(a, L, bt.items);
            LCC_LAUNCH_CHECK();
        }
    }
}

// LCC_TRACE: host-side sections of a round that take > 20 ms (stall hunting)
struct HostProbe {
    bool on = getenv("LCC_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        const double ms = std::chrono::duration<double, std::milli>(now - t).count();
        if (ms > 20.0) fprintf(stderr, "[lcc]       host section '%s' took %.1f ms\n", what, ms);
        t = now;
    }
};

// ---- pulled VertexNeighbors marks (direction-optimising frontier) -------
// A round whose movers are a large part of the graph flags the next frontier
// from the receiving side instead: mark[v] |= OR over u in N(v) of moved[u].
// On a symmetric CSR this is exactly the set the movers' pushes produce
// (every neighbour of a mover), but it costs one short scan per vertex --
// with most vertices moving, the first entries of a row already hold a
// mover -- instead of one random byte store per entry of every mover's row.
// At config 5 those stores fell out of the 126 MB L2 next to the 520 MB
// (label, mass) image and came back as read-modify-write DRAM traffic.
// Head: thread per vertex, the row's first PULL_HEAD entries (independent
// loads); rows not settled there go to a queue that k_pull_rest scans a warp
// per row with early exit.  The moved flags (n bytes) are kept in L2.
constexpr int PULL_HEAD = 4;
__global__ void __launch_bounds__(256) k_pull_head(const int64_t* __restrict__ indptr,
                                                   const int32_t* __restrict__ indices,
                                                   const uint8_t* __restrict__ moved, uint8_t* __restrict__ mark,
                                                   int64_t n, int32_t* __restrict__ rest,
                                                   unsigned long long* __restrict__ nrest) {
    const uint64_t pol_s = policy_evict_first(), pol_k = policy_evict_last();
    const unsigned lane = lane_id();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < n; base += stride) {
        const int64_t v = base + lane;
        bool queue = false;
        if (v < n && !mark[v]) {  // deferred movers are in already
            const int64_t s = indptr[v], d = indptr[v + 1] - s;
            int32_t u[PULL_HEAD];
#pragma unroll
            for (int j = 0; j < PULL_HEAD; ++j) u[j] = j < d ? ld_stream_i32(indices + s + j, pol_s) : -1;
            uint32_t hit = 0;
#pragma unroll
            for (int j = 0; j < PULL_HEAD; ++j) {
                if (u[j] >= 0) {
                    uint16_t m;
                    asm volatile("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(m) : "l"(moved + u[j]), "l"(pol_k));
                    hit |= m;
                }
            }
            if (hit) mark[v] = 1;
            else queue = d > PULL_HEAD;
        }
        const unsigned q = __ballot_sync(FULL, queue);
        if (q) {
            unsigned long long at = 0;
            if (lane == (unsigned)(__ffs(q) - 1)) at = atomicAdd(nrest, (unsigned long long)__popc(q));
            at = __shfl_sync(FULL, at, __ffs(q) - 1);
            if (queue) rest[at + __popc(q & ((1u << lane) - 1u))] = (int32_t)v;
        }
    }
}
__global__ void __launch_bounds__(256) k_pull_rest(const int64_t* __restrict__ indptr,
                                                   const int32_t* __restrict__ indices,
                                                   const uint8_t* __restrict__ moved, uint8_t* __restrict__ mark,
                                                   const int32_t* __restrict__ rest,
                                                   const unsigned long long* __restrict__ nrest) {
    const uint64_t pol_s = policy_evict_first(), pol_k = policy_evict_last();
    const unsigned lane = lane_id();
    const int64_t nq = (int64_t)*nrest;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = (((int64_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); i < nq; i += warps) {
        const int32_t v = rest[i];
        const int64_t end = indptr[v + 1];
        for (int64_t e0 = indptr[v] + PULL_HEAD; e0 < end; e0 += 32) {
            const int64_t e = e0 + lane;
            uint16_t m = 0;
            if (e < end) {
                const int32_t u = ld_stream_i32(indices + e, pol_s);
                asm volatile("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(m) : "l"(moved + u), "l"(pol_k));
            }
            if (__ballot_sync(FULL, m != 0)) {
                if (lane == 0) mark[v] = 1;
                break;
            }
        }
    }
}

// side streams for concurrent bin kernels (one set per device, created once)
struct SideStreams {
    cudaStream_t st[NBINS];
    cudaEvent_t fork;
    cudaEvent_t join[NBINS];
};
inline SideStreams& side_streams() {
    static SideStreams per_dev[16];
    static bool made[16] = {false};
    int dev = 0;
    LCC_CUDA(cudaGetDevice(&dev));
    SideStreams& ss = per_dev[dev & 15];
    if (!made[dev & 15]) {
        for (int i = 0; i < NBINS; ++i) {
            LCC_CUDA(cudaStreamCreateWithFlags(&ss.st[i], cudaStreamNonBlocking));
            LCC_CUDA(cudaEventCreateWithFlags(&ss.join[i], cudaEventDisableTiming));
        }
        LCC_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
        made[dev & 15] = true;
    }
    return ss;
}

// ---- eager kernel loading ----------------------------------------------
// Under CUDA's lazy module loading (the default) a kernel is loaded at its
// first launch, and that load waits for the kernels already running: the
// first round that meets a not-yet-loaded bin kernel runs its concurrent
// bins one after another instead of together.  The asynchronous schedule
// depends on that interleaving -- measured on config 4: a first clustering
// after others in the same process reached 268K-310K instead of 333K, and
// 333K with CUDA_MODULE_LOADING=EAGER.  So every kernel a round may launch
// is loaded (cudaFuncGetAttributes) before its first round starts.
// LCC_MARKBITS=1: the kernels' n-bit neighbour map into the caller's byte mask
// (deferred movers stored their own byte directly)
__global__ void k_bits_to_mask(const unsigned* __restrict__ bits, int64_t n, uint8_t* mark) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
        if ((bits[v >> 5] >> (v & 31)) & 1u) mark[v] = 1;
}

template <class F>
void load_fn(F f) {
    cudaFuncAttributes at;
    LCC_CUDA(cudaFuncGetAttributes(&at, f));
}
template <class WT, bool ASYNC, bool KI>
void preload_ki() {
    load_fn(k_isolated<ASYNC, KI>);
    load_fn(k_tiny<WT, ASYNC, KI>);
    load_fn(k_small<WT, ASYNC, KI>);
    load_fn(k_window<WT, ASYNC, KI>);
    load_fn(k_group<WT, ASYNC, KI, 1, 256, 8, 4, 6>);
    load_fn(k_group<WT, ASYNC, KI, 1, 1024, 8, 8, 3>);
    load_fn(k_group<WT, ASYNC, KI, 4, 2048, 4, 4, 2>);
    load_fn(k_group<WT, ASYNC, KI, 4, 4096, 2, 8, 3>);
    load_fn(k_group<WT, ASYNC, KI, 8, 8192, 1, 4>);
    load_fn(k_group<WT, ASYNC, KI, 32, B5_CAP, 1, 4>);
    load_fn(k_large_score<WT, ASYNC, KI>);
    load_fn(k_large_decide<WT, ASYNC, KI>);
    if constexpr (!WLoad<WT>::fsum) {
        load_fn(k_hub_bucket<WT, ASYNC, KI>);
        load_fn(k_hub_decide<WT, ASYNC, KI>);
    }
}
template <class WT, bool ASYNC>
void preload_round_kernels() {
    static bool done[16] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (done[dev & 15]) return;
    preload_ki<WT, ASYNC, false>();
    preload_ki<WT, ASYNC, true>();
    load_fn(k_large_insert<WT, ASYNC>);
    if constexpr (!WLoad<WT>::fsum) load_fn(k_hub_scatter<WT, ASYNC>);
    load_fn(k_large_mark);
    load_fn(k_pull_head);
    load_fn(k_pull_rest);
    load_fn(k_bits_to_mask);
    load_fn(k_pack32);
    load_fn(k_unpack32);
    load_fn(k_codes);
    load_fn(k_degrees_of);
    load_fn(k_mass_to_u32);
    load_fn(k_mass_from_u32);
    load_fn(k_pack_lk);
    load_fn(k_labels_in);
    load_fn(k_labels_out);
    load_fn(k_bin_count);
    load_fn(k_bin_scatter);
    done[dev & 15] = true;
}

template <class WT, bool ASYNC>
int64_t run_round(const lcc_graph& g, const double* k, double lam, int32_t* C, double* K,
                  const int32_t* frontier, int64_t nF, int deg_threshold, int chunks, int32_t* D,
                  uint8_t* moved, uint8_t* mark, RoundStats* st, cudaStream_t s, const AsyncDamp* damp) {
    const int64_t n = g.n;
    preload_round_kernels<WT, ASYNC>();
    // LCC_L2_FETCH=<bytes> (tuning): the L2's DRAM fetch granularity during
    // the round (cudaLimitMaxL2FetchGranularity); restored afterwards
    static const int l2f = getenv("LCC_L2_FETCH") ? atoi(getenv("LCC_L2_FETCH")) : 0;
    size_t l2f_old = 0;
    if (l2f) {
        LCC_CUDA(cudaDeviceGetLimit(&l2f_old, cudaLimitMaxL2FetchGranularity));
        LCC_CUDA(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)l2f));
    }
    struct L2Restore {
        size_t v;
        ~L2Restore() { if (v) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, v); }
    } l2restore{l2f ? l2f_old : 0};
    HostProbe hprobe;
    if (!ASYNC) LCC_CUDA(cudaMemcpyAsync(D, C, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, s));
    LCC_CUDA(cudaMemsetAsync(moved, 0, n, s));
    if (mark) LCC_CUDA(cudaMemsetAsync(mark, 0, n, s));

    // bin boundaries: warp paths below the degree threshold, CTA paths above
    // (the paper's sequential-vs-parallel hash-table switch)
    // bins: 0 isolated | 1 deg<=8 thread per vertex | 2 ..32 warp windows |
    //       3 optional edge windows | 4-5 warp per vertex up to the threshold |
    //       6 ..1023 4 warps (2K slots) | 7 ..2048 4 warps (4K slots) |
    //       8 ..4096 8 warps | 9 ..large_min 32 warps |
    //       10 hubs (bucketed shared-memory tables)
    // LCC_WINDOW=0 / LCC_LARGE_MIN (env): tuning knobs for the bin shapes only
    // measured on B200 (R-MAT s24): per-vertex warp groups beat the window
    // kernel by ~5%, and CTA groups beat the L2 hub path up to 10240
    const char* ew = getenv("LCC_WINDOW");
    const bool use_window = ew && ew[0] == '1';
    const char* el = getenv("LCC_LARGE_MIN");
    const int64_t large_min = el ? std::max<int64_t>(2048, atoll(el)) : MED_MAX;
    // degree_threshold: warp-per-vertex accumulation below it (the paper's
    // "sequential" path), CTA-cooperative tables from it on ("parallel hash
    // table"); clamped to the warp-table capacity.
    const int64_t Tg = std::min<int64_t>(std::max<int64_t>(deg_threshold, SMALL_MAX + 1), 513);
    int64_t Tw = std::min<int64_t>(std::max<int64_t>(deg_threshold, SMALL_MAX + 1), WIN_W);
    if (!use_window || 2 * n > (1LL << LABEL_BITS)) Tw = SMALL_MAX + 1;  // window keys need ids < 2^27
    int P = 1;
    if (ASYNC && chunks > 0) P = chunks;
    else if (ASYNC) {  // ~4M / F sub-rounds, at most 64 (small graphs need the ordering:
                       // 4 sub-rounds on a 4K-vertex R-MAT drove the objective negative);
                       // chunks < 0: at least -chunks (driver: rounds after the first)
        const int64_t f = std::max<int64_t>(nF, 1);
        P = (int)std::max<int64_t>(1, std::min<int64_t>(64, ((1LL << 22) + f - 1) / f));
        // and no sub-round larger than a wave of LCC_WAVE vertices (default
        // 4M; 0 = off).  One 65M-vertex wave (config 5) let millions of
        // vertices decide on the same stale state: objective 6.90M against
        // the CPU parallel-async oracle's 7.45M (-7.4%); 4M-vertex waves
        // with the bins concurrent inside each: 7.43-7.44M (-0.1%), and the
        // clustering got faster (fewer rounds and levels).  Config 4 (one
        // 16.8M wave was 333K): 305-306K, CPU 303.4K.
        static const int64_t wave = getenv("LCC_WAVE") ? atoll(getenv("LCC_WAVE")) : (1LL << 22);
        if (wave > 0) P = std::max<int>(P, (int)std::min<int64_t>(64, (f + wave - 1) / wave));
        if (chunks < 0) P = std::max(P, -chunks);
    }
    BinEdges be;
    const char* et = getenv("LCC_TINY");  // 0: the warp-window kernel takes degrees 1..32 too
    const int64_t tiny_max = (et && et[0] == '0') ? 0 : TINY_MAX;
    // Small frontiers run as up to 64 ordered sub-rounds of small kernels
    // whose device-side latency dominates: there, neighbouring bins share a
    // kernel (isolated vertices ride in the thread-per-vertex bin -- same
    // arithmetic at degree 0 -- and each pair of table bins takes the larger
    // table), four kernels fewer per sub-round.  LCC_MERGE_BINS=0 disables.
    const char* emb = getenv("LCC_MERGE_BINS");
    const bool merge = P > 1 && nF < (1 << 18) && !(emb && emb[0] == '0');
    be.hi[0] = (merge && tiny_max > 0) ? -1 : 0;  // isolated vertices: only the fresh-singleton option
    be.hi[1] = tiny_max;          // thread per vertex
    be.hi[2] = SMALL_MAX;         // warp-packed windows
    be.hi[3] = Tw - 1;
    be.hi[4] = std::max<int64_t>(be.hi[3], std::min<int64_t>(128, Tg - 1));
    be.hi[5] = std::max<int64_t>(be.hi[4], Tg - 1);
    be.hi[6] = std::max<int64_t>(be.hi[5], std::min<int64_t>(1023, large_min));
    be.hi[7] = std::min<int64_t>(2048, large_min);
    be.hi[8] = std::min<int64_t>(4096, large_min);
    be.hi[9] = std::min<int64_t>(MED_MAX, large_min);
    be.hi[10] = INT64_MAX;
    if (merge) {  // empty bins 4, 6, 8: their vertices go to bins 5, 7, 9
        be.hi[4] = be.hi[3];
        be.hi[6] = be.hi[5];
        be.hi[8] = be.hi[7];
    }

    if (hprobe.on && getenv("LCC_TRACE_SYNC")) {  // device work queued before this round
        LCC_CUDA(cudaStreamSynchronize(s));
        hprobe.mark("prior device work");
    }
    Buf<int32_t> lists(std::max<int64_t>(nF, 1), s);
    hprobe.mark("alloc lists");
    std::vector<int64_t> binstart;
    Buf<unsigned long long> dcnt(4, s);  // [edges, movers, deferred, hub-table overflow]
    LCC_CUDA(cudaMemsetAsync(dcnt.get(), 0, sizeof(unsigned long long) * 4, s));
    unsigned long long* dmoved = dcnt.get() + 1;
    const int64_t ntiles = std::max<int64_t>((nF + BIN_TILE - 1) / BIN_TILE, 1);
    Buf<int64_t> tcnt(NBINS * ntiles + 1, s), tbase(NBINS * ntiles + 1, s);
    unsigned long long hc[NBINS + 1];
    // integer masses (KI kernels): decided here, confirmed by the bin sync.
    // Only for rounds whose frontier is a sizeable part of the graph (the
    // image costs ~n * 36 bytes of traffic per round); LCC_KINT=0 disables.
    const int64_t klen = ASYNC ? 2 * n : n;
    const char* eki = getenv("LCC_KINT");
    const bool try_ki = nF > 0 && 8 * nF >= n && !(eki && eki[0] == '0');
    Buf<uint32_t> Ki;
    Buf<unsigned long long> kchk;
    unsigned long long hk[4] = {0, 0, 0, 0};  // sum of masses, not-integral flag, largest mass or k_v, set codes
    // codes of a packed round (BMArgs::code): built next to the mass image so
    // that their count reaches the host with the bin partition's sync.
    // LCC_CODES=0 disables; LCC_CODES_MIN_PCT: least share of set codes (default 90)
    static const bool codes_on = !(getenv("LCC_CODES") && getenv("LCC_CODES")[0] == '0');
    static const int codes_min_pct = getenv("LCC_CODES_MIN_PCT") ? atoi(getenv("LCC_CODES_MIN_PCT")) : 90;
    Buf<unsigned> codes;
    float kconv_ms = 0.f;
    cudaEvent_t kev[2] = {nullptr, nullptr};
    if (try_ki) {
        for (auto& e : kev) LCC_CUDA(cudaEventCreateWithFlags(&e, cudaEventDefault));
        Ki.alloc(KS * klen, s);  // interleaved: (label, mass) pairs -- masses at odd words, labels below
        kchk.alloc(4, s);
        LCC_CUDA(cudaMemsetAsync(kchk.get(), 0, sizeof(unsigned long long) * 4, s));
        LCC_CUDA(cudaEventRecord(kev[0], s));
        k_mass_to_u32<<<grid_for(klen, 256), 256, 0, s>>>(K, klen, k, n, Ki.get() + (KS - 1), kchk.get(),
                                                           reinterpret_cast<unsigned*>(kchk.get() + 1),
                                                           reinterpret_cast<unsigned*>(kchk.get() + 2));
        LCC_LAUNCH_CHECK();
        if (LCC_CODES && ASYNC && LCC_ILV && codes_on && chunks < 0) {
            codes.alloc((n + 7) / 8, s);
            k_codes<<<grid_for((n + 7) / 8, 256), 256, 0, s>>>(C, Ki.get() + (KS - 1), n, codes.get(), kchk.get() + 3);
            LCC_LAUNCH_CHECK();
        }
        LCC_CUDA(cudaEventRecord(kev[1], s));
        LCC_CUDA(cudaMemcpyAsync(hk, kchk.get(), sizeof(hk), cudaMemcpyDeviceToHost, s));
    }
    if (nF > 0) {
        k_bin_count<<<(unsigned)ntiles, BIN_THREADS, 0, s>>>(g.indptr, frontier, nF, be, ntiles, tcnt.get(), dcnt.get());
        LCC_LAUNCH_CHECK();
        LCC_CUDA(cudaMemsetAsync(tcnt.get() + NBINS * ntiles, 0, sizeof(int64_t), s));
        exclusive_sum(tcnt.get(), tbase.get(), NBINS * ntiles + 1, s);
        hprobe.mark("count + scan enqueue");
        k_bin_scatter<<<(unsigned)ntiles, BIN_THREADS, 0, s>>>(g.indptr, frontier, nF, be, ntiles, tbase.get(),
                                                               lists.get());
        LCC_LAUNCH_CHECK();
        // bin b occupies [tbase[b*ntiles], tbase[(b+1)*ntiles]) of `lists`
        std::vector<int64_t> hb(NBINS + 1);
        for (int b = 0; b <= NBINS; ++b)
            LCC_CUDA(cudaMemcpyAsync(&hb[b], tbase.get() + (int64_t)b * ntiles, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        LCC_CUDA(cudaMemcpyAsync(&hc[NBINS], dcnt.get(), sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
        hprobe.mark("scatter + D2H enqueue");
        LCC_CUDA(cudaStreamSynchronize(s));
        for (int b = 0; b < NBINS; ++b) hc[b] = (unsigned long long)(hb[b + 1] - hb[b]);
        binstart.assign(hb.begin(), hb.end());
        hprobe.mark("bin partition (incl. device wait)");
    } else {
        for (int b = 0; b <= NBINS; ++b) hc[b] = 0;
        binstart.assign(NBINS + 1, 0);
    }
    // Edge-heavy small frontiers (a few 10K coarse hubs with 10^8 entries):
    // the vertex-count rule above gives them 64 ordered sub-rounds of a few
    // hundred CTAs each, which the launch tails dominate.  LCC_SUB_EDGES (A/B
    // knob, 0 = off): no sub-round smaller than that many entries, but never
    // fewer than 8 sub-rounds, and only for frontiers of >= 2^26 entries.
    {
        static const int64_t sub_edges = getenv("LCC_SUB_EDGES") ? atoll(getenv("LCC_SUB_EDGES")) : (1LL << 26);
        const int64_t fe = (int64_t)hc[NBINS];
        if (ASYNC && chunks <= 0 && sub_edges > 0 && fe >= (1LL << 26) && P > 8) {
            const int cap = (int)std::max<int64_t>(8, (fe + sub_edges - 1) / sub_edges);
            P = std::min(P, std::max(cap, chunks < 0 ? -chunks : 1));
        }
    }
    const bool ki = try_ki && hk[1] == 0 && hk[0] < (1ull << 31);
    if (try_ki) LCC_CUDA(cudaEventElapsedTime(&kconv_ms, kev[0], kev[1]));
    const bool dmp = ASYNC && damp && damp->prev_moved && mark;  // deferral needs the fused frontier
    // neighbour marks: pushed by the movers inside the kernels (default), or
    // pulled after them (k_pull_*, LCC_PULL=1; whole graphs only -- a shard's
    // CSR holds only its own rows).  Measured on B200, round 1 from
    // singletons: pull 120.4 vs push 115.3 ms (config 5), 12.0 vs 10.7 ms
    // (config 4), config-5 clustering 4.2-4.8 vs 3.0 s -- the asynchronous
    // kernels run slower without the mark stores between vertices (the same
    // interleaving effect as round 1's unfused-mark test), more than the
    // stores cost.
    const char* epl = getenv("LCC_PULL");
    const bool pull = mark && nF > 0 && !(g.flags & LCC_GRAPH_PARTIAL_ROWS) && epl && epl[0] == '1';
    // packed (label, mass) words for the group bins (integer masses only)
    Buf<unsigned long long> LK;
    const bool use_lk = ki && LCC_LK && (!ASYNC || LCC_LK_ASYNC) && !WLoad<WT>::fsum && nF > 0;
    if (use_lk) LK.alloc(n, s);
    const bool ilv = ki && LCC_ILV;
    int32_t* CK = ilv ? reinterpret_cast<int32_t*>(Ki.get()) : nullptr;  // labels at even, masses at odd
    BMArgs a{g.indptr, g.indices, g.weights, k, lam, ilv ? CK : C,
             ki ? (void*)(Ki.get() + (KS - 1)) : (void*)K, D, moved, dmoved, (int32_t)n, mark,
             dmp ? damp->prev_moved : nullptr, dmp ? damp->salt : 0u, dcnt.get() + 2, use_lk ? LK.get() : nullptr,
             ilv ? 2 : 1, mark, nullptr, -1, (int32_t)KS, 0, 0.0};
    if (pull) a.mark = nullptr;  // neighbour marks pulled after the kernels
    // Packed words (see BMArgs): asynchronous integer-mass rounds whose labels
    // (ids < 2n) leave at least 4 bits of a 32-bit word for the masses, and
    // whose masses and vertex weights start at no more than half the field
    // (a join that would pass the field's top is refused, like a failed
    // commit check).  LCC_PACK32=0 (env) keeps the interleaved 64-bit image.
    Buf<uint32_t> W32;
    int pk_lb = 0;
    {
        const char* epk = getenv("LCC_PACK32");
        int lb = std::max(1, bit_width((uint64_t)std::max<int64_t>(klen - 1, 1)));
        if (const char* eb = getenv("LCC_PACK32_BITS")) lb = std::max(lb, atoi(eb));  // tests: a narrow mass field
        const unsigned cap = lb <= 28 ? (1u << (32 - lb)) - 1u : 0u;
        if (LCC_PACK32 && ASYNC && ilv && !use_lk && !(epk && epk[0] == '0') && cap >= 15u && hk[2] <= cap / 2) {
            pk_lb = lb;
            W32.alloc(klen, s);
            a.C = reinterpret_cast<int32_t*>(W32.get());
            a.K = W32.get();
            a.cs = 1;
            a.ks = 1;
            a.ksh = lb;
            a.lm = (int32_t)((1u << lb) - 1u);
            a.kmax = (double)(cap - 1u);
        }
        // codes: packed or interleaved words alike (async integer-mass rounds)
        // (not in a level's very first round from singletons at the finest
        // level -- chunks == 0 -- where most vertices move and the codes would
        // all be cleared on the way: config 5 round 1 151 vs 119 ms)
        if (LCC_CODES && ASYNC && ilv && !use_lk && chunks < 0 && codes.get() && (double)hk[3] * 100.0 >= (double)codes_min_pct * (double)n)
            a.code = codes.get();
    }
    Buf<unsigned> mbits;
    if (LCC_MARKBITS == 1 && a.mark) {
        mbits.alloc((n + 31) / 32, s);
        LCC_CUDA(cudaMemsetAsync(mbits.get(), 0, sizeof(unsigned) * ((n + 31) / 32), s));
        a.mbits = mbits.get();
    }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    LCC_CUDA(cudaEventCreateWithFlags(&ev0, cudaEventDefault));
    LCC_CUDA(cudaEventCreateWithFlags(&ev1, cudaEventDefault));
    const long long launches0 = launch_counter();
    float kms = 0.f;

    WindowPlan wp;
    if (hc[3] > 0) plan_windows(g.indptr, lists.get() + binstart[3], (int64_t)hc[3], wp, s);
    const int64_t nL = (int64_t)hc[NBINS - 1];
    // The bins are independent within a (sub-)round -- sync reads a frozen
    // state and writes disjoint D entries; async tolerates any interleaving --
    // so their latency-bound kernels run concurrently on side streams
    // (fork/join with events) instead of back to back.
    // With ordered async sub-rounds (P > 1, small frontiers) the bins stay in
    // order on the caller's stream: the interleaving is what breaks symmetry
    // on small graphs (measured on the config-1 SBM).
    SideStreams& ss = side_streams();
    // (frontiers of a wave or more: the bins also overlap inside each ordered
    // sub-round -- measured better objectives than bin-ordered sub-rounds
    // there, 7.44M vs 7.40M on config 5; LCC_SUBCONC=0/1 forces it off/on)
    const char* esc = getenv("LCC_SUBCONC");
    const bool concurrent = P == 1 || (esc ? (esc[0] == '1' && nF >= (1 << 20))
                                           : nF >= (1 << 22));
    LCC_CUDA(cudaEventRecord(ev0, s));
    if (pk_lb) {  // timed with the kernels
        k_pack32<<<grid_for(klen, 256), 256, 0, s>>>(C, Ki.get() + (KS - 1), n, klen, pk_lb, W32.get());
        LCC_LAUNCH_CHECK();
    } else if (ilv) {
        k_labels_in<<<grid_for(n, 256), 256, 0, s>>>(C, n, CK);
        LCC_LAUNCH_CHECK();
    }
    if (use_lk) {
        k_pack_lk<<<grid_for(n, 256), 256, 0, s>>>(C, Ki.get() + (KS - 1), n, LK.get());
        LCC_LAUNCH_CHECK();
    }
    auto launch_all = [&](auto ki_tag) {
    constexpr bool KI = decltype(ki_tag)::value;
    for (int j = 0; j < P; ++j) {
        LCC_CUDA(cudaEventRecord(ss.fork, s));
        int used = 0;
        auto next_stream = [&]() -> cudaStream_t {
            if (!concurrent) return s;
            cudaStream_t t = ss.st[used++];
            LCC_CUDA(cudaStreamWaitEvent(t, ss.fork, 0));
            return t;
        };
        // (diagnostics: LCC_LAUNCH_DELAY_US stalls the host after every bin
        // launch; LCC_HUBS_LAST launches the hub bin after the others)
        static const int dly = getenv("LCC_LAUNCH_DELAY_US") ? atoi(getenv("LCC_LAUNCH_DELAY_US")) : 0;
        static const bool hubs_last = getenv("LCC_HUBS_LAST") && getenv("LCC_HUBS_LAST")[0] == '1';
        if (j == 0 && nL > 0 && !hubs_last) run_large<WT, ASYNC, KI>(a, g, lists.get() + binstart[NBINS - 1], nL,
                                                       reinterpret_cast<unsigned*>(dcnt.get() + 3), next_stream());
        for (int b = 0; b < NBINS - 1; ++b) {
            if (dly) std::this_thread::sleep_for(std::chrono::microseconds(dly));
            const int64_t nb = (int64_t)hc[b];
            if (nb == 0) continue;
            const int32_t* list = lists.get() + binstart[b];
            if (b == 3) {
                if (wp.nwin * (j + 1) / P > wp.nwin * j / P)
                    launch_window<WT, ASYNC, KI>(a, list, wp, wp.nwin * j / P, wp.nwin * (j + 1) / P, next_stream());
                continue;
            }
            const int64_t lo = nb * j / P, hi = nb * (j + 1) / P;
            if (hi <= lo) continue;
            cudaStream_t t = next_stream();
            if (b == 0) {
                k_isolated<ASYNC, KI><<<grid_for(hi - lo, 256, 8), 256, 0, t>>>(a, list, lo, hi);
                LCC_LAUNCH_CHECK();
            } else if (b == 1) {
                k_tiny<WT, ASYNC, KI><<<grid_for(hi - lo, 256, 8), 256, 0, t>>>(a, list, lo, hi);
                LCC_LAUNCH_CHECK();
            } else if (b == 2) {
                const int64_t warps = (hi - lo + 31) / 32;
                k_small<WT, ASYNC, KI><<<grid_for(warps * 32, SMALL_THREADS, 8), SMALL_THREADS, 0, t>>>(a, list, lo, hi);
                LCC_LAUNCH_CHECK();
            } else {
                launch_bin<WT, ASYNC, KI>(b - 2, a, list, lo, hi, t);
            }
        }
        if (j == 0 && nL > 0 && hubs_last) run_large<WT, ASYNC, KI>(a, g, lists.get() + binstart[NBINS - 1], nL,
                                                      reinterpret_cast<unsigned*>(dcnt.get() + 3), next_stream());
        for (int i = 0; i < used; ++i) {
            LCC_CUDA(cudaEventRecord(ss.join[i], ss.st[i]));
            LCC_CUDA(cudaStreamWaitEvent(s, ss.join[i], 0));
        }
    }
    };
    if (ki) launch_all(std::true_type{});
    else launch_all(std::false_type{});
    if (a.mbits) {
        k_bits_to_mask<<<grid_for(n, 256), 256, 0, s>>>(a.mbits, n, mark);
        LCC_LAUNCH_CHECK();
    }
    if (pull) {
        Buf<int32_t> rest(n, s);
        Buf<unsigned long long> nrest(1, s);
        LCC_CUDA(cudaMemsetAsync(nrest.get(), 0, sizeof(unsigned long long), s));
        k_pull_head<<<grid_for(n, 256, 16), 256, 0, s>>>(g.indptr, g.indices, moved, mark, n, rest.get(), nrest.get());
        LCC_LAUNCH_CHECK();
        k_pull_rest<<<num_sms() * 8, 256, 0, s>>>(g.indptr, g.indices, moved, mark, rest.get(), nrest.get());
        LCC_LAUNCH_CHECK();
    }
    if (pk_lb) {
        k_unpack32<<<grid_for(klen, 256), 256, 0, s>>>(W32.get(), n, klen, pk_lb, C, K);
        LCC_LAUNCH_CHECK();
    } else if (ki && ASYNC) {  // async moves updated the image: back to fp64 K (and the labels to C)
        k_mass_from_u32<<<grid_for(klen, 256), 256, 0, s>>>(Ki.get() + (KS - 1), klen, K);
        LCC_LAUNCH_CHECK();
        if (ilv) {
            k_labels_out<<<grid_for(n, 256), 256, 0, s>>>(CK, n, C);
            LCC_LAUNCH_CHECK();
        }
    }
    hprobe.mark("launches");
    LCC_CUDA(cudaEventRecord(ev1, s));
    unsigned long long hm = 0, hp = 0, hov = 0;
    LCC_CUDA(cudaMemcpyAsync(&hm, dmoved, sizeof(hm), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaMemcpyAsync(&hp, dcnt.get() + 2, sizeof(hp), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaMemcpyAsync(&hov, dcnt.get() + 3, sizeof(hov), cudaMemcpyDeviceToHost, s));
    LCC_CUDA(cudaStreamSynchronize(s));
    if (hov) throw CudaError("hub bucket table overflow (LCC_HUB_BUCKETS=0 selects the global-table path)");
    hprobe.mark("kernels (device wait)");
    LCC_CUDA(cudaEventElapsedTime(&kms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    for (auto& e : kev)
        if (e) cudaEventDestroy(e);
    kms += kconv_ms;  // the mass image is part of the round's kernel time
    const float kms_large = 0.f;
    if (st) {
        st->vertices += nF;
        st->edges += (int64_t)hc[NBINS];
        st->moved += (int64_t)hm;
        st->n_small += (int64_t)(hc[0] + hc[1] + hc[2]);
        for (int b = 3; b < NBINS - 1; ++b) st->n_medium += (int64_t)hc[b];
        st->n_large += nL;
        st->ms_kernels += (double)kms + (double)kms_large;
        st->launches += launch_counter() - launches0;
    }
    return (int64_t)(hm + hp);  // deferred movers keep the iteration loop going
}

}  // namespace

int64_t best_moves_round(const lcc_graph& g, const double* k, double lam, int32_t* C, double* K,
                         const int32_t* frontier, int64_t nF, int schedule, int deg_threshold,
                         int async_chunks, int32_t* D, uint8_t* moved, uint8_t* mark, RoundStats* st,
                         cudaStream_t s, const AsyncDamp* damp) {
    LCC_REQUIRE(g.n >= 0 && g.n < (1LL << 30), "vertex count out of range");
    LCC_REQUIRE(schedule == LCC_SYNC || schedule == LCC_ASYNC, "unknown schedule");
    LCC_REQUIRE(schedule == LCC_ASYNC || D != nullptr, "sync schedule needs D");
    LCC_REQUIRE(async_chunks >= -64, "async_chunks out of range");
    if (g.n == 0) return 0;
    // NULL = all vertices unless the caller asked for an empty frontier
    // (nF == 0: D = C, moved / mark cleared, no kernels)
    const bool as = schedule == LCC_ASYNC;
    switch (g.weights ? g.wtype : LCC_W_NONE) {
        case LCC_W_NONE:
            return as ? run_round<WNone, true>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, mark, st, s, damp)
                      : run_round<WNone, false>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, mark, st, s, damp);
        case LCC_W_F32:
            return as ? run_round<float, true>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, mark, st, s, damp)
                      : run_round<float, false>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, mark, st, s, damp);
        case LCC_W_F64:
            return as ? run_round<double, true>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, mark, st, s, damp)
                      : run_round<double, false>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, mark, st, s, damp);
        case LCC_W_U32:
            // integer sums in 32-bit slots: every per-vertex sum <= 2 * total weight
            LCC_REQUIRE(2.0 * g.total_weight < 4294967296.0, "uint32 weights need 2 * total_weight < 2^32");
            return as ? run_round<uint32_t, true>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, mark, st, s, damp)
                      : run_round<uint32_t, false>(g, k, lam, C, K, frontier, nF, deg_threshold, async_chunks, D, moved, mark, st, s, damp);
        default:
            throw Invalid("unknown weight dtype");
    }
}

}  // namespace lcc
